# ncu --set full of the adjoint kernel of one step (usage: bash scripts/gpu/ncu_ga.sh c3)
c=${1:-c3}
python scripts/ncu_step.py --config $c > gpurun_out/ncu_ga_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bp_gather \
    -o gpurun_out/ncu_ga python scripts/ncu_step.py --config $c > gpurun_out/ncu_ga.log 2>&1
echo "rc=$?"
python scripts/ncu_metrics.py gpurun_out/ncu_ga.ncu-rep
ncu -i gpurun_out/ncu_ga.ncu-rep --page raw --csv > gpurun_out/ncu_ga_raw.csv
rm -f gpurun_out/ncu_ga.ncu-rep
