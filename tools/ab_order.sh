python -m pytest tests/test_gpu_parity.py -q -x -k "mv_gala2" 2>&1 | tail -2
for o in 1; do for b in 8 32; do
GALA_MAC2_ORDER=$o python bench.py --steps 20 --warmup 3 --batch $b --no-cpu-baseline > gpurun_out/abo_${o}_${b}.json 2> gpurun_out/abo_${o}_${b}.err
python -c "
import json; d=json.load(open('gpurun_out/abo_${o}_${b}.json'))
print('order $o batch $b value', d['value'], 'mac2', d['kernel_breakdown_ms_per_step'].get('k_gala_mac2'), 'e', d['kernel_breakdown_ms_per_step'].get('k_gala_e'), d['roofline']['frac'])"
done; done
