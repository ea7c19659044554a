cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/t17.log
for a in "u3 gate_up 1" "i5 gate_up 1" "f6e3m2 gate_up 1" "u8 gate_up 1" "u3 qkv 1" "u3 down 1" "u8 qkv 1" "u3 gate_up 16" "u8 gate_up 16"; do timeout 120 python tools/prof_one.py $a >> gpurun_out/p17.txt 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extra --no-c5 > gpurun_out/b17.json 2> gpurun_out/b17.err
cat gpurun_out/t17.log; grep "us=" gpurun_out/p17.txt; grep -i error gpurun_out/p17.txt | head -3; tail -2 gpurun_out/b17.err; python -c "import json;d=json.loads(open('gpurun_out/b17.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])"
