cd $GRAFT_REPO_ROOT
for n in 4 6 8 12 16 24; do TL_TCD_NS=$n timeout -s KILL 100 python tools/prof_graph.py u4 gate_up 1 3 u8 gate_up 1 3 u4 o 1 3 2>&1 | grep -v Warn | sed "s/^/ns=$n /"; done
