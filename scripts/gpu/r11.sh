python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py -m gpu -x -q -k "not slow" 2>&1 | tail -2
CFG=c1 bash scripts/gpu/ab_env.sh base NCSG_ORB_NW=8 "NCSG_GA_CHUNKS=6"
