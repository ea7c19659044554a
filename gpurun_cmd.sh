cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3; do for f in u8 u7 f8e4m3 u3; do for l in down gate_up qkv o; do timeout 60 python tools/grid_sweep.py $f $l 1 1 0 >> gpurun_out/gv40.txt 2>&1 || echo "FAIL $f $l" >> gpurun_out/gv40.txt; done; done; done
timeout 300 compute-sanitizer --tool memcheck python tools/run_shape.py u8 28672 8192 1 1 > gpurun_out/san40.txt 2>&1; tail -3 gpurun_out/san40.txt
grep -c "us=" gpurun_out/gv40.txt; grep "FAIL" gpurun_out/gv40.txt | sort | uniq -c
