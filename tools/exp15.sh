cd $GRAFT_REPO_ROOT
for d in 0 1 4 5; do TL_TCD_DBG=$d timeout -s KILL 100 python tools/prof_graph.py u4 gate_up 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done
./tools/mma_probe | grep "TS N= 16"
