timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -x -q --timeout 120 2>&1 | tail -25
