cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q -k tcs 2>&1 | tail -3
timeout -s KILL 200 python tools/prof_graph.py u3 o 1 3 u4 8192x1024 1 3 u4 o 1 3 u4 gate_up 1 3 u3 gate_up 1 3 i5 gate_up 1 3 f6e3m2 gate_up 1 3 u8 gate_up 1 3 u4 gate_up 16 3 f6e3m2 gate_up 16 3 2>&1 | grep -v Warn
timeout -s KILL 60 python tools/trace_tcd.py u4 gate_up 1 2>&1 | tail -30
