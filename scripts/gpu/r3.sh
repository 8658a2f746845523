python -m pytest tests/test_cpp_api.py tests/test_gpu_solver.py tests/test_gpu_ncstomo.py -m gpu -x -q -k "not slow and not c4 and not c5" 2>&1 | tail -15
