cd $GRAFT_REPO_ROOT
for f in i5 u3 u4 f6e3m2 u8 i4 u5; do timeout -s KILL 30 python tools/prof_graph.py $f gate_up 1 3 2>&1 | grep -v Warn || echo "$f HANG/FAIL"; done
