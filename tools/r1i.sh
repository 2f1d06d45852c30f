python tools/bench_configs.py > gpurun_out/configs_r1i.jsonl 2> gpurun_out/configs_r1i.err || tail -20 gpurun_out/configs_r1i.err
python tools/bench_resnet18.py > gpurun_out/resnet_r1i.jsonl 2> gpurun_out/resnet_r1i.err || tail -20 gpurun_out/resnet_r1i.err
python -c "
import json
for l in open('gpurun_out/configs_r1i.jsonl'):
    d=json.loads(l); b=d.get('batch') or {}
    print(d['config'], round(d['ms_per_layer'],5), d['correct'], json.dumps(d['roofline']), json.dumps(b.get('roofline')), b.get('ms_per_layer'), b.get('correct'))
"
tail -1 gpurun_out/resnet_r1i.jsonl
