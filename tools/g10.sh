python -m pytest tests -m gpu -q -x > gpurun_out/g10_pytest.log 2>&1; tail -2 gpurun_out/g10_pytest.log
python bench.py --no-cpu-baseline --steps 20 > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err || tail -5 gpurun_out/g10_bench.err
python -c "
import json; d=json.load(open('gpurun_out/g10_bench.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'roof', d['roofline']['bound'], d['roofline']['frac'], 'layer', d['roofline']['layer']['frac'])
print(json.dumps(d['kernel_breakdown_ms_per_step']))"
