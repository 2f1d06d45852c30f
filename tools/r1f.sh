python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/bench_sharded_conv.py > gpurun_out/sharded_conv.json 2> gpurun_out/sharded_conv.err || tail -20 gpurun_out/sharded_conv.err
cat gpurun_out/sharded_conv.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/bench_resnet18.py > gpurun_out/resnet_r1f.jsonl 2> gpurun_out/resnet_r1f.err || tail -20 gpurun_out/resnet_r1f.err
tail -1 gpurun_out/resnet_r1f.jsonl
