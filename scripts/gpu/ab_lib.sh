# A/B of variant libraries on the C3 bench: bash scripts/gpu/ab_lib.sh base name1 name2 ...
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="NCSG_LIB=_variants/$v/libncsg.so"; fi
  env $L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --config ${CFG:-c3} > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
done
