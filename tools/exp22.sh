cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q -k "tcs or chain" 2>&1 | tail -2
for f in u4 u3 i5 f6e3m2 u8; do timeout -s KILL 30 python tools/prof_graph.py $f gate_up 1 3 $f o 1 3 2>&1 | grep -v Warn || echo "$f HANG/FAIL"; done
timeout -s KILL 60 python tools/trace_tcd.py u4 gate_up 1 2>&1 | grep -A8 "group 0 iter"
