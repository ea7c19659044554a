cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 60 python tools/prof_graph.py u4 8192x1024 1 3 u4 o 1 3 u3 qkv 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn
timeout -s KILL 60 python tools/trace_pdl.py u4 8192x1024 2>&1 | tail -15 | head -6
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null > gpurun_out/b24.json
