cd $GRAFT_REPO_ROOT
for f in u3 u4 i5 f6e3m2 u8; do for l in o gate_up; do python tools/prof_one.py $f $l 1 1; python tools/prof_one.py $f $l 1 3; done; done 2>&1 | grep -v Warn
python tools/trace_tcs.py u4 gate_up 1 > gpurun_out/trace_u4.txt 2>&1
