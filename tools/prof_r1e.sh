# round-1 evidence pass 2: bench line, reference arm, launch list, ncu of the batched first-Add
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r1e.log 2>&1
python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r1e.json 2> gpurun_out/ref_r1e.err
CMD="python bench.py --steps 2 --warmup 3 --batch 32 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv $CMD > gpurun_out/ncu_launch_r1e.log 2>&1
CFG3_BATCH=16 ncu --set full --clock-control none --import-source on -k regex:"k_kg_accumulate" -s 1 -c 1 -o gpurun_out/prof_kgacc_r1e python tools/bench_configs.py cfg3 > gpurun_out/ncu_kgacc_r1e.log 2>&1
tail -1 gpurun_out/smoke_r1e.log; cut -c1-300 gpurun_out/bench_r1e.json; cut -c1-300 gpurun_out/ref_r1e.json; ls -la gpurun_out/*.ncu-rep
