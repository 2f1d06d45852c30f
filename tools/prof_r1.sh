set -e
CMD="python bench.py --steps 1 --warmup 1 --batch 2 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd -s 60 -c 1 -o gpurun_out/prof_ntt $CMD > gpurun_out/ncu_ntt.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:k_ks_accum -s 2 -c 1 -o gpurun_out/prof_ks $CMD > gpurun_out/ncu_ks.log 2>&1 || true
ls -la gpurun_out
