NCSG_LIB=_variants/le3/libncsg.so python -m pytest tests/test_gpu_ops.py -m gpu -x -q -k "fft or mask or solve" 2>&1 | tail -2
for c in c2 c3 c1 c5; do CFG=$c bash scripts/gpu/ab_lib.sh base le3; done
