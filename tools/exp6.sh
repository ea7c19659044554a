cd $GRAFT_REPO_ROOT
for l in 8192x1024 o gate_up; do timeout -s KILL 60 python tools/trace_tcd.py u4 $l 1 2>&1 | grep -v Warn; done
