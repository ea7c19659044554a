cd $GRAFT_REPO_ROOT
./tools/mma_probe
for d in 0 1 2 4 7; do echo "dbg=$d"; for f in u4 u8; do for l in o gate_up; do TL_TCD_DBG=$d timeout -s KILL 60 python tools/prof_one.py $f $l 1 3; done; done 2>&1 | grep -v Warn; done
