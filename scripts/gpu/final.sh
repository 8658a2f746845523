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
# summaries on the box (gpurun_out/ travels back only under 64 MiB): the
# per-config csv/json (and C3's raw page) go to gpurun_out/profiles/, the
# reports themselves are dropped
mkdir -p gpurun_out/profiles
for c in c3 c1 c2 c5 c4; do
  [ -f gpurun_out/ncu_$c.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/ncu_$c.ncu-rep r2 $c > /dev/null &&
    cp profiles/r2_ncu_$c.csv profiles/ncu_$c.json gpurun_out/profiles/
done
ncu -i gpurun_out/ncu_c3.ncu-rep --page raw --csv > gpurun_out/profiles/r2_ncu_c3_raw.csv 2>/dev/null
rm -f gpurun_out/ncu_*.ncu-rep
NCSG_OUT=gpurun_out/r2_shard_projection.json python scripts/shard_step_time.py c3 c4 c5 2>&1 | tail -3
