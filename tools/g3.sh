# round-2 (session 3) measurement: bench line at the key-folded default, bench contract test, launch list,
# one ncu --set full capture of k_gala_kf (one 256-input tile)
mkdir -p gpurun_out
python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err || tail -20 gpurun_out/g3_bench.err
python -m pytest tests/test_bench_contract.py -q > gpurun_out/g3_contract.log 2>&1; tail -2 gpurun_out/g3_contract.log
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/g3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/g3_ncu_launch.log 2>&1
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_gala_kf|k_gala_dq" -c 2 \
    -o gpurun_out/prof_kf_r2 -f python tools/time_fc.py > gpurun_out/g3_ncu_full.log 2>&1
echo done
