cd $GRAFT_REPO_ROOT
for fp in 1 3; do TL_FORCE_PATH=$fp timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-e2e --no-cpu > gpurun_out/b_fp$fp.json 2> gpurun_out/b_fp$fp.err; tail -2 gpurun_out/b_fp$fp.err; done
