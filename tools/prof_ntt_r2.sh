#!/usr/bin/env bash
# ncu --set full of the FC step's NTT-class kernels (config 2, B = 32): digit INTT, digit NTTs into the
# other primes, the ModDown INTT and the ModDown NTT + combine.
cd "$(dirname "$0")/.."
B=32 python tools/time_fc.py > gpurun_out/r2_ntt_pre.log 2>&1
B=32 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
    -k regex:"k_digits_intt|k_digits_perm|k_ntt_inv|k_moddown" -c 4 \
    -o gpurun_out/prof_ntt_r2 -f python tools/time_fc.py > gpurun_out/r2_ncu_ntt.log 2>&1
echo done
