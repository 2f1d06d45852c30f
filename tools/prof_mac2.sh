set -e
CMD="python bench.py --steps 2 --warmup 3 --batch 32 --no-cpu-baseline"
$CMD > gpurun_out/plain_mac2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gala_mac2" -s 3 -c 1 -o gpurun_out/prof_mac2_v2 $CMD > gpurun_out/ncu_mac2_v2.log 2>&1
