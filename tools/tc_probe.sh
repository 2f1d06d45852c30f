# k_gala_tc role isolation: which unit paces a position (experiment builds, no correctness)
for f in "-DGTC_NO_A" "-DGTC_NO_A -DGTC_NO_B" "-DGTC_NO_A -DGTC_NO_EPI" "-DGTC_NO_A -DGTC_NO_B -DGTC_NO_EPI" "-DGTC_NO_B -DGTC_NO_EPI"; do
  GALA_NVCC_EXTRA="$f" python -c "from paper_2105_01827_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "$f: $(python tools/time_fc.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["k_gala_tc"])')"
done
for f in "-DGTC_NO_A -DGTC_NO_B -DGTC_NO_EPI" "-DGTC_NO_A -DGTC_NO_B -DGTC_NO_EPI -DGTC_MMA_REPEAT=2" "-DGTC_NO_A -DGTC_NO_B -DGTC_NO_EPI -DGTC_MMA_REPEAT=4"; do
  GALA_NVCC_EXTRA="$f" python -c "from paper_2105_01827_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "$f: $(python tools/time_fc.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["k_gala_tc"])')"
done
