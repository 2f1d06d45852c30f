for v in 1 0; do
  GALA_MAC3=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_$v.json 2>gpurun_out/ab3_$v.err || tail -3 gpurun_out/ab3_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab3_$v.json')); b=d['kernel_breakdown_ms_per_step']; print('MAC3=$v', d['value'], b.get('k_gala_mac3'), b.get('k_gala_mac2'))"
done
