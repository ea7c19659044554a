cd $GRAFT_REPO_ROOT
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tcd_kernel -s 3 -c 1 -o gpurun_out/tcd_u4_gateup python tools/prof_one.py u4 gate_up 1 3 > gpurun_out/ncu16.log 2>&1
tail -3 gpurun_out/ncu16.log
