# per-config ncu --set full capture of one NCS step: bash scripts/gpu/ncu_cfg.sh c1 c2 ...
for c in "$@"; do
  python scripts/ncu_step.py --config $c > gpurun_out/ncu_plain_$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o gpurun_out/ncu_$c python scripts/ncu_step.py --config $c > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
