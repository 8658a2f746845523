python -m pytest tests/test_gpu_ops.py -m gpu -x -q 2>&1 | tail -2
bash scripts/gpu/ab_lib.sh base t24m3 t16m3 t16m4
CFG=c4 STEPS=5 bash scripts/gpu/ab_lib.sh base t24m3
