# launch list (layer kernels only) of the bench command; ncu --set full of k_gala_kf (one 256-input tile) and
# of the NTT-class kernels of the same step
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_gala_kf$|k_gala_dq|k_digits|k_ks_|k_moddown|k_ntt_inv|k_giant|k_sub_plain|k_encode" \
    --log-file gpurun_out/g4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/g4_ncu_launch.log 2>&1
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"^k_gala_kf$" -c 1 \
    -o gpurun_out/prof_kf_r2 -f python tools/time_fc.py > gpurun_out/g4_ncu_kf.log 2>&1
B=256 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
    -k regex:"k_digits_intt|k_digits_perm|k_ntt_inv|k_moddown|k_ks_mac" -c 5 \
    -o gpurun_out/prof_ntt_r2b -f python tools/time_fc.py > gpurun_out/g4_ncu_ntt.log 2>&1
echo done
