python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for b in 32; do
python bench.py --steps 20 --warmup 3 --batch $b --no-cpu-baseline > gpurun_out/abB_${b}.json 2> gpurun_out/abB_${b}.err || tail -3 gpurun_out/abB_${b}.err
python -c "
import json; d=json.load(open('gpurun_out/abB_${b}.json'))
print('batch $b baby', d['config']['bsgs_baby'], 'value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], json.dumps(d['kernel_breakdown_ms_per_step']))"
done
