# adjoint chunk-count sweep at a config: bash scripts/gpu/ga_sweep.sh c3 9 10 11 12 ...
cfg=$1; shift
for c in "$@"; do
  NCSG_GA_CHUNKS=$c python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ga_$c.log 2>&1
  python - $c <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/ga_{sys.argv[1]}.log').read().strip().splitlines()[-1])
print('chunks', sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
done
