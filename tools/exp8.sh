cd $GRAFT_REPO_ROOT
for d in 0 8 40 47; do echo dbg=$d; TL_TCD_DBG=$d timeout -s KILL 60 python tools/trace_tcd.py u4 gate_up 1 2>&1 | tail -40 | head -12; TL_TCD_DBG=$d timeout -s KILL 60 python tools/prof_graph.py u4 gate_up 1 3 | grep -v Warn; done
