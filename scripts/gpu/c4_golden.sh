# C4 golden on the GPU box's host cores (the oracle port, OpenMP): writes
# gpurun_out/c4_full.npz; copy it to tests/golden/ afterwards.
nproc; free -g | head -2; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
N=$(nproc)
if [ "$N" -ge 24 ]; then
  T=$N; [ "$T" -gt 128 ] && T=128
  NCS_GOLDEN_OUT=gpurun_out/c4_full.npz timeout ${C4_TIMEOUT:-3300} python tests/golden/make_c4_golden.py $T
else
  echo "too few cores ($N) for the C4 golden here"
fi
