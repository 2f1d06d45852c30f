# evidence pass at the default bench batch (96): launch list, all configs, ResNet-18, reference arm
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_r1f.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv $CMD > gpurun_out/ncu_launch_r1f.log 2>&1
python tools/bench_configs.py > gpurun_out/configs_r1f.jsonl 2> gpurun_out/configs_r1f.err
python tools/bench_resnet18.py > gpurun_out/resnet_r1f.jsonl 2> gpurun_out/resnet_r1f.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r1f.json 2> gpurun_out/ref_r1f.err
tail -1 gpurun_out/resnet_r1f.jsonl | cut -c1-200; cut -c1-200 gpurun_out/ref_r1f.json; wc -l gpurun_out/launches_r1f.csv gpurun_out/configs_r1f.jsonl
