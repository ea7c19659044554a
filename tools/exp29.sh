cd $GRAFT_REPO_ROOT
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tcd_kernel -s 3 -c 1 -o gpurun_out/tcd_u3_gateup python tools/prof_one.py u3 gate_up 1 3 > /dev/null 2>&1
ls -la gpurun_out/tcd_u3_gateup.ncu-rep
