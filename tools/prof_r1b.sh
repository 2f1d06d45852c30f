set -e
python __graft_entry__.py > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
CMD="python bench.py --steps 2 --warmup 1 --batch 2 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_digits_perm -s 4 -c 1 -o gpurun_out/prof_perm_r1b $CMD > gpurun_out/ncu_perm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ks_mac -s 4 -c 1 -o gpurun_out/prof_mac_r1b $CMD > gpurun_out/ncu_mac.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_digits_intt -s 4 -c 1 -o gpurun_out/prof_intt_r1b $CMD > gpurun_out/ncu_intt.log 2>&1
