# quick GPU iteration: one focused test file (fail fast), per-layer decode timings, optional full suite
# + bench line.  TESTS=<file> FMTS="u3 i5" LAYERS="gate_up qkv" M=1 FULL=1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-q}
if [ -n "$TESTS" ]; then timeout -s KILL 600 python -m pytest $TESTS -q -x 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_pytest.log; fi
for fmt in ${FMTS:-u3 i5 f6e3m2 u8 u1 u4 i8}; do for layer in ${LAYERS:-gate_up qkv o down}; do
  timeout -s KILL 60 python tools/prof_one.py $fmt $layer ${M:-1} 2>&1 | tail -1
done; done > gpurun_out/${TAG}_layers.txt 2>&1
cat gpurun_out/${TAG}_layers.txt
if [ -n "$FULL" ]; then
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_pytest_gpu.log; tail -c 300 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
fi
