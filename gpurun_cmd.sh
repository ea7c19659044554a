cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in 0; do echo "dbg=$d" >> gpurun_out/gs30.txt; TL_TC2_DBG=$d timeout 200 python tools/grid_sweep.py u3 gate_up 128 2 112 148 >> gpurun_out/gs30.txt 2>&1;  TL_TC2_DBG=$d timeout 200 python tools/grid_sweep.py u3 qkv 128 2 80 120 148 >> gpurun_out/gs30.txt 2>&1; TL_TC2_DBG=$d timeout 200 python tools/grid_sweep.py u3 o 128 2 64 128 148 >> gpurun_out/gs30.txt 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -x -k "batched or tc" 2>&1 | tail -2 >> gpurun_out/gs30.txt; cat gpurun_out/gs30.txt
