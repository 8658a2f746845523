python -m pytest tests/test_cpp_api.py -m gpu -q 2>&1 | tail -3
