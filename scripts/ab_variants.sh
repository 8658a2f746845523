for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then L=""; else L="NCSG_LIB=_variants/$v/libncsg.so"; fi
  env $L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  echo "$v $(grep -o "\"forward\": [0-9.]*\|\"adjoint\": [0-9.]*\|\"fft_[a-z_0-9]*\": [0-9.]*" gpurun_out/ab_$v.log | tr "\n" " ") $(grep -o '"value": [0-9.]*' gpurun_out/ab_$v.log | head -1)"
done
