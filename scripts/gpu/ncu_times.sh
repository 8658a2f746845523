# per-kernel durations of one NCS step (warm caches, no clock control): bash scripts/gpu/ncu_times.sh c2 c3 ...
for c in "$@"; do
  python scripts/ncu_step.py --config $c > gpurun_out/nt_plain_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off \
      --csv --log-file gpurun_out/nt_$c.csv python scripts/ncu_step.py --config $c > gpurun_out/nt_$c.log 2>&1
  echo "$c rc=$?"
  python - $c <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/nt_{sys.argv[1]}.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=0
for r in rows[1:]:
    v=float(r[vi]); tot+=v; print(f'  {r[ki][:40]:40s} {v/1000:8.2f} us')
print(f'  total {tot/1000:.2f} us')
PY
done
