cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/t22.log
for a in "u3 qkv 128" "u3 o 128" "u3 gate_up 128" "u3 down 128" "i5 gate_up 128" "f6e3m2 gate_up 128" "u8 gate_up 128" "u8 qkv 128" "u3 gate_up 64" "u3 gate_up 32"; do timeout 120 python tools/prof_one.py $a >> gpurun_out/p22.txt 2>&1; done
cat gpurun_out/t22.log; grep "us=" gpurun_out/p22.txt; grep -i error gpurun_out/p22.txt | head -3
