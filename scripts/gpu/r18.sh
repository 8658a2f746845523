python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py -m gpu -x -q -k "not slow" 2>&1 | tail -2
bash scripts/gpu/ab_env.sh base
CFG=c5 bash scripts/gpu/ab_env.sh base
CFG=c2 bash scripts/gpu/ab_env.sh base
