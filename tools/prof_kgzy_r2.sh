#!/usr/bin/env bash
# ncu --set full of the config-4 schedule-2 kernels (k_kg_zy, k_kg_tc) of one post-mask layer
set -e
cd "$(dirname "$0")/.."
python tools/time_kg_forms.py > gpurun_out/r2_kgforms_pre_ncu.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_kg_zy|k_kg_tc$" -c 2 \
    -o gpurun_out/prof_kgzy_r2 -f python tools/time_kg_forms.py > gpurun_out/ncu_kgzy_r2.log 2>&1
