cd $GRAFT_REPO_ROOT
for d in 0 8 16 31; do echo dbg=$d; TL_TCD_DBG=$d timeout -s KILL 100 python tools/prof_graph.py u4 8192x1024 1 3 u4 8192x2048 1 3 u4 o 1 3 u4 gate_up 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn; done
timeout -s KILL 100 python tools/prof_graph.py u4 8192x1024 1 1 u4 8192x2048 1 1 2>&1 | grep -v Warn
