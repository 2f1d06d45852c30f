for sp in 0 1; do for v in 0 5 6 7 8; do
if [ $sp = 1 ]; then export GALA_NO_SPLIT60=1; fi
GALA_MAC2_VAR=$v python bench.py --steps 15 --warmup 3 --batch 32 --no-cpu-baseline > gpurun_out/abg.json 2> gpurun_out/abg.err || tail -3 gpurun_out/abg.err
python -c "
import json; d=json.load(open('gpurun_out/abg.json'))
print('nosplit=$sp var=$v value', d['value'], 'mac2', d['kernel_breakdown_ms_per_step']['k_gala_mac2'])"
done; done
GALA_MAC2_VAR=5 python -m pytest tests/test_gpu_parity.py -q -x -k "mv_gala2" 2>&1 | tail -1
GALA_MAC2_VAR=7 python -m pytest tests/test_gpu_parity.py -q -x -k "mv_gala2" 2>&1 | tail -1
