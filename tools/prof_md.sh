set -e
CMD="python tools/time_fc.py"
$CMD > gpurun_out/plain_md.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_moddown|k_digits_perm" -s 6 -c 2 -o gpurun_out/prof_md $CMD > gpurun_out/ncu_md.log 2>&1
