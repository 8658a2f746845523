# A/B of environment switches on the C3 bench: bash scripts/gpu/ab_env.sh "ENV1=a" "ENV2=b" ...
# ("base" = no extra environment)
for v in "$@"; do
  if [ "$v" = base ]; then E=""; else E="$v"; fi
  env $E python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --config ${CFG:-c3} > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
done
