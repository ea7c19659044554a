cd $GRAFT_REPO_ROOT
timeout -s KILL 60 python tools/prof_one.py u4 o 1 3 2>&1 | tail -3
timeout -s KILL 300 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q -k tcs 2>&1 | tail -8
for f in u3 u4 i5 f6e3m2 u8; do for l in qkv o gate_up down; do timeout -s KILL 60 python tools/prof_one.py $f $l 1 3; done; done 2>&1 | grep -v Warn
for f in u4 f6e3m2; do for l in o gate_up; do timeout -s KILL 60 python tools/prof_one.py $f $l 16 3; done; done 2>&1 | grep -v Warn
