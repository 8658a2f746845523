timeout 1500 python -m pytest tests -m gpu -x -q -k "not slow" 2>&1 | tail -6
