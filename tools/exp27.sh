cd $GRAFT_REPO_ROOT
for d in 0 256 4; do TL_TCD_DBG=$d timeout -s KILL 60 python tools/prof_graph.py i5 qkv 16 3 f6e3m2 qkv 16 3 u8 down 16 3 f6e3m2 down 16 3 i5 qkv 1 3 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done
