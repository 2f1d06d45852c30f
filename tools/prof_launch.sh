set -e
CMD="python bench.py --steps 2 --warmup 3 --batch 32 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv $CMD > gpurun_out/ncu_launch_r1h.log 2>&1
