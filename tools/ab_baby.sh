for bb in 32 64 16; do
  python bench.py --steps 20 --warmup 3 --batch 32 --no-cpu-baseline --baby $bb > gpurun_out/abb_$bb.json 2>gpurun_out/abb_$bb.err || tail -3 gpurun_out/abb_$bb.err
  python -c "
import json; d=json.load(open('gpurun_out/abb_$bb.json')); print('baby=$bb', d['value'], json.dumps(d['kernel_breakdown_ms_per_step']))"
done
