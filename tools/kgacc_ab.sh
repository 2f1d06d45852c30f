# config-3 first-Add tile / accumulator A/B (k_kg_accumulate): GALA_KGACC="img,odt", GALA_KGACC_PP=0|1
run() { CFG3_BATCH=16 python tools/bench_configs.py cfg3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['batch']; print('$1', round(d['ms_per_layer']*1e3,1), round(b['ms_per_layer']*1e3,1), b['roofline']['frac'], b['breakdown_ms_per_layer']['k_kg_accumulate'], d['breakdown_ms']['k_kg_accumulate'])"; }
run default
GALA_KGACC=2,1 GALA_KGACC_PP=1 run "2,1 pp"
GALA_KGACC=1,2 GALA_KGACC_PP=1 run "1,2 pp"
GALA_KGACC=1,4 GALA_KGACC_PP=1 run "1,4 pp"
GALA_KGACC=2,2 GALA_KGACC_PP=1 run "2,2 pp"
