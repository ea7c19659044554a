cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/t3.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
for a in "u3 gate_up 1" "i5 gate_up 1" "f6e3m2 gate_up 1" "u8 gate_up 1" "u3 qkv 1" "u3 qkv 128" "u3 gate_up 128" "f6e3m2 gate_up 128"; do timeout 120 python tools/prof_one.py $a >> gpurun_out/p3.txt 2>&1; done
tail -3 gpurun_out/t3.log; cat gpurun_out/p3.txt; tail -2 gpurun_out/b3.err
