cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q -k tcs 2>&1 | tail -2
for f in u4 u3 i5 f6e3m2 u8; do for l in gate_up o; do timeout -s KILL 30 python tools/prof_graph.py $f $l 1 3 $f $l 1 1 2>&1 | grep -v Warn || echo "$f $l HANG/FAIL"; done; done
