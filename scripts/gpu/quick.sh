# quick GPU check: operator parity + C3 bench phases (usage: bash scripts/gpu/quick.sh [pytest-args])
python -m pytest tests/test_gpu_ops.py -m gpu -x -q "$@" 2>&1 | tail -3
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/quick.log 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/quick.log').read().strip().splitlines()[-1])
print('value', round(d['value'],1), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
