python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_words.py -q -x > gpurun_out/g11_parity.txt 2>&1; tail -2 gpurun_out/g11_parity.txt
B=256 python tools/time_fc.py
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"^k_gala_kf$" -c 1 \
    -o gpurun_out/prof_kf_r2b -f python tools/time_fc.py > gpurun_out/g11_ncu_kf.log 2>&1
echo done
