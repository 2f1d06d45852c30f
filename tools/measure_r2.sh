#!/usr/bin/env bash
# Round-2 evidence pass on one B200 (each ncu capture after its command exited 0 without ncu):
#   bench line (default flags), reference arm, layer-kernel launch list of the bench command,
#   ncu --set full of k_gala_kf (one 256-input tile) and of the FC step's NTT-class kernels,
#   per-config and ResNet-18 side benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/m2_bench.json 2> gpurun_out/m2_bench.err || tail -5 gpurun_out/m2_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m2_ref.json 2> gpurun_out/m2_ref.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_gala_kf$|k_gala_dq|k_digits|k_ks_|k_moddown|k_ntt_inv|k_giant|k_sub_plain|k_encode" \
    --log-file gpurun_out/m2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/m2_ncu_launch.log 2>&1
B=256 python tools/time_fc.py > gpurun_out/m2_time_fc.json 2>&1
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"^k_gala_kf$" -c 1 \
    -o gpurun_out/prof_kf_m2 -f python tools/time_fc.py > gpurun_out/m2_ncu_kf.log 2>&1
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
    -k regex:"k_digits_intt|k_digits_perm|k_ntt_inv|k_moddown|k_ks_mac" -c 5 \
    -o gpurun_out/prof_ntt_m2 -f python tools/time_fc.py > gpurun_out/m2_ncu_ntt.log 2>&1
python tools/bench_configs.py > gpurun_out/m2_configs.jsonl 2> gpurun_out/m2_configs.err
python tools/bench_resnet18.py --net resnet18_224.net > gpurun_out/m2_resnet18_224.jsonl 2> gpurun_out/m2_resnet.err
echo done
