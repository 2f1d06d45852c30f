for opt in "" "--no-tensor-cores"; do
python bench.py --steps 20 --warmup 3 --batch 32 --no-cpu-baseline $opt > gpurun_out/abtc.json 2> gpurun_out/abtc.err || tail -5 gpurun_out/abtc.err
python -c "
import json; d=json.load(open('gpurun_out/abtc.json'))
print('opt=$opt value', d['value'], 'e2e', d['e2e']['value'], d['config']['baby_step_sums'], json.dumps(d['kernel_breakdown_ms_per_step']))"
done
