# ncu of the orbit forward (and adjoint) of one C3 step for the base build and variants
python scripts/ncu_step.py --config c3 > gpurun_out/plain_fwd.log 2>&1 || exit 1
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="NCSG_LIB=_variants/$v/libncsg.so"; fi
  env $L ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"fp_orbit|bp_gather" \
    -o gpurun_out/fwd_$v python scripts/ncu_step.py --config c3 > gpurun_out/ncu_fwd_$v.log 2>&1
  echo "$v rc=$?"
done
