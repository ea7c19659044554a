# ncu --set full of one decode launch, summarised on the box: FMT LAYER M
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
TAG=${TAG:-n}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tcd_kernel} -s 6 -c 1 -o /tmp/ncu/${TAG} python tools/prof_one.py ${FMT:-u3} ${LAYER:-gate_up} ${M:-1} > /dev/null 2> gpurun_out/${TAG}_ncu.err
python tools/ncu_summary.py /tmp/ncu/${TAG}.ncu-rep > gpurun_out/${TAG}.txt 2>&1
ncu -i /tmp/ncu/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
cat gpurun_out/${TAG}.txt
