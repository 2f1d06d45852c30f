# bench line (default flags), reference arm, layer-kernel launch list of the bench command, configs and ResNet-18 side benches
python bench.py > gpurun_out/g12_bench.json 2> gpurun_out/g12_bench.err || tail -5 gpurun_out/g12_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g12_ref.json 2> gpurun_out/g12_ref.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_gala_kf$|k_gala_dq|k_digits|k_ks_|k_moddown|k_ntt_inv|k_giant|k_sub_plain|k_encode" \
    --log-file gpurun_out/g12_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/g12_ncu_launch.log 2>&1
python tools/bench_configs.py > gpurun_out/g12_configs.jsonl 2> gpurun_out/g12_configs.err
python tools/bench_resnet18.py --net resnet18_224.net > gpurun_out/g12_resnet18_224.jsonl 2> gpurun_out/g12_resnet.err
echo done
