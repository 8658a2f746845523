# C4 golden on the GPU box's host cores (the oracle port, OpenMP): writes
# gpurun_out/c4_<iters>.npz (NCS_GOLDEN_ITERS, default the config's 300 ->
# c4_full.npz); copy it to tests/golden/ afterwards.
N=$(nproc); echo "host cores: $N"
IT=${NCS_GOLDEN_ITERS:-300}
OUT=gpurun_out/c4_$IT.npz; [ "$IT" = 300 ] && OUT=gpurun_out/c4_full.npz
NCS_GOLDEN_ITERS=$IT NCS_GOLDEN_OUT=$OUT timeout ${C4_TIMEOUT:-3300} python tests/golden/make_c4_golden.py $N
