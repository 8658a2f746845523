python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py -m gpu -x -q -k "not slow" 2>&1 | tail -3
bash scripts/gpu/ab_env.sh base NCSG_GA_CLUSTER=1 NCSG_GA_CLUSTER=2
