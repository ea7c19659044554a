cd $GRAFT_REPO_ROOT
TL_LIB_PATH=$PWD/abtest/lib_nw6.so timeout -s KILL 600 python -m pytest tests/test_gpu_matmul.py -m gpu -x -q -k "tcs or chain" 2>&1 | tail -1
for lib in "" "$PWD/abtest/lib_nw6.so"; do for i in 1 2; do TL_LIB_PATH=$lib timeout 300 python bench.py --steps 30 --warmup 3 --no-extra --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lib=${lib##*/}', d['value'], d['ms_per_step'])"; done; done
for lib in "" "$PWD/abtest/lib_nw6.so"; do TL_LIB_PATH=$lib timeout -s KILL 60 python tools/prof_graph.py u3 gate_up 1 3 i5 gate_up 1 3 f6e3m2 gate_up 1 3 u8 gate_up 1 3 u3 o 1 3 2>&1 | grep -v Warn | sed "s|^|${lib##*/} |"; done
