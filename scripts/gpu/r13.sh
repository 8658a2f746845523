python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py -m gpu -x -q -k "not slow" 2>&1 | tail -2
for c in c3 c2 c1; do
CFG=$c bash scripts/gpu/ab_env.sh base NCSG_NO_FUSED_FFT=1 NCSG_LIB=_variants/fminb1/libncsg.so
done
