python -m pytest tests/test_gpu_parity.py -q -x -k "mv_gala2" 2>&1 | tail -1
for v in 0 1; do
if [ $v = 1 ]; then export GALA_NO_SPLIT60=1; fi
python bench.py --steps 20 --warmup 3 --batch 32 --no-cpu-baseline > gpurun_out/abs_$v.json 2> gpurun_out/abs_$v.err || tail -3 gpurun_out/abs_$v.err
python -c "
import json; d=json.load(open('gpurun_out/abs_$v.json'))
print('nosplit=$v value', d['value'], 'frac', d['roofline']['frac'], json.dumps(d['kernel_breakdown_ms_per_step'])[:200])"
done
