set -x
python -m pytest tests/test_gpu_ops.py -m gpu -x -q 2>&1 | tail -5
for rq in 8 auto; do
  if [ $rq = auto ]; then unset NCSG_ORB_RQ; else export NCSG_ORB_RQ=$rq; fi
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_rq$rq.log 2>&1
  echo "rq=$rq $(grep -o '"forward": [0-9.]*\|"adjoint": [0-9.]*\|"value": [0-9.]*' gpurun_out/ab_rq$rq.log | head -3 | tr '\n' ' ')"
done
