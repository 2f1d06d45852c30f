python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err || tail -20 gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json'))
print('value', d['value'], 'e2e', json.dumps(d['e2e']))"
