for ch in 1 2 4 8; do
  GALA_MAC2_CH=$ch python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abc_$ch.json 2>gpurun_out/abc_$ch.err || tail -3 gpurun_out/abc_$ch.err
  python -c "
import json; d=json.load(open('gpurun_out/abc_$ch.json')); b=d['kernel_breakdown_ms_per_step']; print('CH=$ch', d['value'], b.get('k_gala_mac2'))"
done
