cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 3 --no-extra --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'])"; done
timeout -s KILL 60 python tools/prof_graph.py u3 gate_up 1 3 i5 gate_up 1 3 f6e3m2 gate_up 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn
