# one GPU session: parity suite, smoke, tcgen05 dispatch probe, bench line, ncu launch list of the bench
# step, ncu --set full of the decode kernel summarised ON the box (the .ncu-rep stays out of gpurun_out:
# the reports of a 180 MB library exceed the 64 MiB copy-back limit)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/ncu
TAG=${TAG:-r2}
timeout -s KILL 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1
if [ -x tools/mma_probe2 ]; then timeout -s KILL 120 tools/mma_probe2 > gpurun_out/${TAG}_mma_probe2.txt 2>&1; fi
timeout -s KILL 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu --no-c5 --no-spectrum > /dev/null 2> gpurun_out/${TAG}_ncu_launch.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tcd_kernel -s 6 -c 1 -o /tmp/ncu/${TAG}_tcd_u3_gateup_m1 python tools/prof_one.py u3 gate_up 1 > /dev/null 2>> gpurun_out/${TAG}_ncu_full.err
python tools/ncu_summary.py /tmp/ncu/${TAG}_tcd_u3_gateup_m1.ncu-rep > gpurun_out/${TAG}_tcd_u3_gateup_m1.txt 2>&1
cat gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_smoke.log gpurun_out/${TAG}_mma_probe2.txt; tail -c 300 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
du -sh gpurun_out
