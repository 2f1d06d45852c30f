#!/usr/bin/env bash
# Round-2 measurement session on one B200: bench line, per-config and ResNet-18 side benches, the
# ncu launch list of the bench command, one ncu --set full capture of the bench's dominant kernels.
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
python tools/bench_configs.py > gpurun_out/r2_configs.jsonl 2> gpurun_out/r2_configs.err
python tools/bench_resnet18.py --net resnet18_224.net > gpurun_out/r2_resnet18_224.jsonl 2> gpurun_out/r2_resnet.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/r2_ncu_launch.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_gala_e_can|k_gala_tc" -c 2 \
    -o gpurun_out/prof_gala_r2 -f python tools/time_fc.py > gpurun_out/r2_ncu_full.log 2>&1
echo done
