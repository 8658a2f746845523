# FFT engine A/B: operator parity, then per-config bench with the old (NCSG_FFT_P2=0) and new passes
python -m pytest tests/test_gpu_ops.py -m gpu -x -q 2>&1 | tail -3
for c in ${CFGS:-c2 c3 c1}; do
  for v in "NCSG_FFT_P2=0" "NCSG_FFT_P2=1" "$@"; do
    env $v python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --config $c > gpurun_out/fab.log 2>&1
    python - "$c $v" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/fab.log').read().strip().splitlines()[-1])
    print(sys.argv[1], 'value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items() if 'fft' in k or 'dual' in k})
except Exception as e:
    print(sys.argv[1], 'FAILED', e); print(open('gpurun_out/fab.log').read()[-1500:])
PY
  done
done
