cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/t31.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b31.json 2> gpurun_out/b31.err
cat gpurun_out/t31.log; tail -2 gpurun_out/b31.err; python - <<'PY'
import json
d=json.loads(open('gpurun_out/b31.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
for x in d['details']: print('M1', x['fmt'], x['layer'], x['us'], x['hbm_frac'])
for x in d['details_extra_M']: print('M%d'%x['M'], x['fmt'], x['layer'], x['us'], x['TFLOPs'], x['tensor_frac_fp16'])
for x in d['details_c5'] or []: print('C5', x)
print(d.get('cpu_baseline'))
PY
