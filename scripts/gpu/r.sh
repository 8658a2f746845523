python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py -m gpu -x -q -k "not slow and not c4 and not c5" 2>&1 | tail -3
bash scripts/gpu/ab_env.sh base NCSG_DUAL_RAY_MAJOR=1
