cd $GRAFT_REPO_ROOT
ARGS=""
for f in u3 u4 i5 f6e3m2 u8; do for l in qkv o gate_up down; do ARGS="$ARGS $f $l 1 1 $f $l 1 3"; done; done
timeout -s KILL 300 python tools/prof_graph.py $ARGS 2>&1 | grep -v Warn
for d in 1 7; do TL_TCD_DBG=$d timeout -s KILL 100 python tools/prof_graph.py u4 o 1 3 u4 gate_up 1 3 u8 gate_up 1 3 2>&1 | grep -v Warn; done
