# bench every config (no CPU baseline / e2e): bash scripts/gpu/allcfg.sh [extra env]
for c in ${CFGS:-c1 c2 c3 c4 c5}; do
  env "$@" python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e --config $c > gpurun_out/all_$c.log 2>&1
  python - $c <<'PY'
import json,sys
try:
    d=json.loads(open(f'gpurun_out/all_{sys.argv[1]}.log').read().strip().splitlines()[-1])
    print(sys.argv[1], 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in d['phases_ms'].items()}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))
except Exception as e:
    print(sys.argv[1], 'FAILED', e); print(open(f'gpurun_out/all_{sys.argv[1]}.log').read()[-2000:])
PY
done
