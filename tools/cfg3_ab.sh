# config-3 A/B: image batch size and the tensor-core first-Add threshold (prints ms per layer and roofline)
for b in 16 32 64; do
  echo "batch $b: $(CFG3_BATCH=$b python tools/bench_configs.py cfg3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); b=d["batch"]; print(round(b["ms_per_layer"]*1e3,1), "us/layer, frac", b["roofline"]["frac"], b["breakdown_ms_per_layer"])')"
done
echo "tc1 batch 16: $(CFG3_BATCH=16 python -c '
import runpy, sys
import paper_2105_01827_b200.conv as c
c.KG1_TC_MIN_BYTES = 0
sys.argv = ["bench_configs.py", "cfg3"]
runpy.run_path("tools/bench_configs.py", run_name="__main__")' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); b=d["batch"] or {}; print(d["ms_per_layer"], b.get("ms_per_layer"), b.get("breakdown_ms_per_layer"), d["breakdown_ms"])')"
