cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "prefill" 2>&1 | tail -4
for M in 256 512 1024 2048 4096 8192; do for pth in 2 4; do timeout 120 python tools/grid_sweep.py u4 gate_up $M $pth 0 2>&1 | grep "us="; done; done
for M in 512 1024 4096; do for pth in 2 4; do timeout 120 python tools/grid_sweep.py u4 qkv $M $pth 0 2>&1 | grep "us="; done; done
