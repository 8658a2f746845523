python -m pytest tests/test_gpu_solver.py -m gpu -q -s -k "seminorm or records or record_every" 2>&1 | grep -E "seminorm|passed|failed|Error|assert" | head -20
