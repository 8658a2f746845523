python -m pytest tests/test_gpu_multi.py tests/test_gpu_ops.py -m gpu -x -q --timeout 200 2>&1 | tail -2
bash scripts/gpu/ab_env.sh base
CFG=c2 bash scripts/gpu/ab_env.sh base
