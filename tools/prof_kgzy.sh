set -e
CMD="python tools/bench_configs.py cfg4"
$CMD > gpurun_out/plain_kgzy.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_kg_zy" -s 2 -c 1 -o gpurun_out/prof_kgzy $CMD > gpurun_out/ncu_kgzy.log 2>&1
