mkdir -p gpurun_out
tools/mma_bench > gpurun_out/g2_mma.txt 2>&1
tools/mma_bench ring > gpurun_out/g2_mma_ring.txt 2>&1
NAMES="base onlyMMA noA noB noE noW" B=256 sh tools/kf_probe.sh > gpurun_out/g2_probe.txt 2>&1
python -m pytest tests -m gpu -q --deselect tests/test_bench_contract.py::test_gpu_arm_line > gpurun_out/g2_pytest.log 2>&1; tail -5 gpurun_out/g2_pytest.log
echo done
