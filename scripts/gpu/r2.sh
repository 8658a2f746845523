python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_c3.log 2>&1; tail -c 3000 gpurun_out/b_c3.log
timeout 1500 bash scripts/gpu/ncu_cfg.sh c3 c1 c2 c5 c4
