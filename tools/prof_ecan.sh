set -e
CMD="python tools/time_fc.py"
$CMD > gpurun_out/plain_ecan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gala_e_can" -s 3 -c 1 -o gpurun_out/prof_ecan_v2 $CMD > gpurun_out/ncu_ecan_v2.log 2>&1
