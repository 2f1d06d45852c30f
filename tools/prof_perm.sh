set -e
CMD="python bench.py --steps 2 --warmup 1 --batch 8 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_digits_perm -s 2 -c 1 -o gpurun_out/prof_perm_sf $CMD > gpurun_out/ncu_perm.log 2>&1
