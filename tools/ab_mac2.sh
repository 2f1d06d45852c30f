for cb in 1 2 4; do
  GALA_MAC2_CB=$cb python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$cb.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$cb.json')); print('CB=$cb', d['value'], d['kernel_breakdown_ms_per_step'].get('k_gala_mac2'))"
done
