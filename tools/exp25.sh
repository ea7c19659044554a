cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 60 python tools/prof_graph.py u4 8192x1024 1 3 u3 o 1 3 u3 qkv 16 3 u3 gate_up 16 3 u8 gate_up 1 3 2>&1 | grep -v Warn
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null > gpurun_out/b25.json
