# round-1 evidence pass (no profiler): smoke, default bench line, reference arm, all configs, ResNet-18
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r1d.log 2>&1
python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r1d.json 2> gpurun_out/ref_r1d.err
python tools/bench_configs.py > gpurun_out/configs_r1d.jsonl 2> gpurun_out/configs_r1d.err
python tools/bench_resnet18.py > gpurun_out/resnet_r1d.jsonl 2> gpurun_out/resnet_r1d.err
tail -1 gpurun_out/smoke_r1d.log; cat gpurun_out/bench_r1d.json | cut -c1-600; tail -2 gpurun_out/resnet_r1d.jsonl | cut -c1-300
