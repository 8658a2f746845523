# table-mode vs direct adjoint at several configs: bash scripts/gpu/wt_cfgs.sh c1 c5 c4
for c in "$@"; do
  for m in 1 0; do
    NCSG_GA_WTAB=$m python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/wtc.log 2>&1
    python - "$c wtab=$m" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/wtc.log').read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
  done
done
