mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; tail -5 gpurun_out/g1_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err || tail -20 gpurun_out/g1_bench.err
for b in 96 256; do B=$b python tools/time_fc.py > gpurun_out/g1_timefc_$b.json 2>&1; done
GALA_FC_KF=0 B=96 python tools/time_fc.py > gpurun_out/g1_timefc_96_nokf.json 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --batch 256 > gpurun_out/g1_bench256.json 2> gpurun_out/g1_bench256.err || tail -20 gpurun_out/g1_bench256.err
echo done
