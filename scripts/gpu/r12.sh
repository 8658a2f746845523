python -m pytest tests/test_gpu_multi.py -m gpu -q 2>&1 | tail -3
for c in c3 c5; do
NCSG_BENCH_GLOO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --config $c > gpurun_out/multi_$c.log 2>&1
echo "$c rc=$?"; tail -c 1500 gpurun_out/multi_$c.log
done
