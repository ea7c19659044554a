cd $GRAFT_REPO_ROOT
for d in 0 128; do TL_TCD_DBG=$d timeout -s KILL 60 python tools/prof_graph.py u4 8192x1024 1 3 u4 o 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done
for d in 0 128; do TL_TCD_DBG=$d timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg=$d bench', d['value'], d['ms_per_step'])"; done
