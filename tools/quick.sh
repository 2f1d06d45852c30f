# quick GPU iteration: parity tests + bench line + kernel breakdown
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err || tail -20 gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'layer frac', d['roofline']['layer']['frac'], 'peak', d['roofline']['peak'])
print(json.dumps(d['kernel_breakdown_ms_per_step']))"
