python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor_core or gala2" 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err || tail -20 gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json'))
print('value', d['value'], 'e2e', d['e2e']['value'])
print(json.dumps(d['kernel_breakdown_ms_per_step']))"
