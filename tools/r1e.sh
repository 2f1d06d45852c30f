python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_kg" 2>&1 | tail -2
CFG3_BATCH=16 python tools/bench_configs.py cfg3 > gpurun_out/cfg3_t.json 2> gpurun_out/cfg3.err || tail -20 gpurun_out/cfg3.err
python -c "
import json
d=json.load(open('gpurun_out/cfg3_t.json')); print('single', round(d['ms_per_layer'],4), 'batch', json.dumps(d['batch']))
"
