# one GPU session: parity suite, smoke, bench line, ncu launch list of the bench step, ncu --set full of tcd
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-e2e --no-cpu > /dev/null 2> gpurun_out/ncu_launch.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tcd_kernel -s 40 -c 1 -o gpurun_out/tcd_full python bench.py --steps 2 --warmup 1 --no-extra --no-e2e --no-cpu > /dev/null 2> gpurun_out/ncu_full.err
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 300 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
