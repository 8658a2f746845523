# Round-end measurement set (into gpurun_out/): bench lines per config, the
# reference arm, the ncu launch list of the default bench command, per-config
# ncu --set full captures of one NCS step, serialized per-kernel durations,
# and the per-rank shard projection.  GPU tests: scripts/gpu/full.sh.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err
for c in c1 c2 c4 c5; do
  python bench.py --steps 20 --warmup 5 --config $c --no-cpu-baseline > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
done
python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_launches.log 2>&1
bash scripts/gpu/ncu_times.sh c1 c2 c3 c5 > gpurun_out/final_ncu_times.log 2>&1
timeout 1500 bash scripts/gpu/ncu_cfg.sh c3 c1 c2 c5 c4
NCSG_OUT=gpurun_out/r2_shard_projection.json python scripts/shard_step_time.py c3 c4 c5 2>&1 | tail -3
