cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 60 python tools/prof_graph.py i5 qkv 16 3 u8 down 16 3 i5 qkv 1 3 u3 o 1 3 2>&1 | grep -v Warn
timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step']); [print(r['fmt'],r['layer'],r['M'],r['us']) for r in d['details_extra_M'] if r['M']==16]"
