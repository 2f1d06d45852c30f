set -e
CMD="python bench.py --steps 2 --warmup 1 --batch 8 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gala_mac2|k_gala_e|k_digits_perm|k_moddown" -s 8 -c 4 -o gpurun_out/prof_r1c $CMD > gpurun_out/ncu_full.log 2>&1
