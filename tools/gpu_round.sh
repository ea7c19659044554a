# one GPU session (round 2): parity suite, smoke, bench line, ncu launch list of the bench step (time + DRAM
# bytes per launch), ncu --set full of the decode kernel (u3 gate_up M=1) and the batched kernel (u3 gate_up M=128)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu --no-c5 --no-spectrum > /dev/null 2> gpurun_out/${TAG}_ncu_launch.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tcd_kernel -s 6 -c 1 -o gpurun_out/${TAG}_tcd_u3_gateup_m1 python tools/prof_one.py u3 gate_up 1 > /dev/null 2>> gpurun_out/${TAG}_ncu_full.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 6 -c 1 -o gpurun_out/${TAG}_tc2_u3_gateup_m128 python tools/prof_one.py u3 gate_up 128 > /dev/null 2>> gpurun_out/${TAG}_ncu_full.err
cat gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_smoke.log; tail -c 400 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
