cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-e2e --no-cpu > gpurun_out/b_pdl.json 2> gpurun_out/b_pdl.err; tail -2 gpurun_out/b_pdl.err
for f in u4 u3 u8; do timeout -s KILL 30 python tools/prof_graph.py $f gate_up 1 3 $f o 1 3 2>&1 | grep -v Warn || echo "$f HANG/FAIL"; done
