# table-mode adjoint sweep: bash scripts/gpu/wt_sweep.sh c3 "PF=4 CH=12" "PF=8 CH=6" ...
cfg=$1; shift
for v in "$@"; do
  eval $v
  env NCSG_GA_WT_PF=${PF:-4} ${CH:+NCSG_GA_CHUNKS=$CH} python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/wt.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/wt.log').read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
  unset PF CH
done
