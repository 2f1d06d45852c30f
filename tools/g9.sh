NAMES="a4b2 a3b3 a5b1 j4a8b4 j4a10b2 a4b2only" B=256 sh tools/kf_probe.sh > gpurun_out/g9_probe.txt 2>&1
NST=8 ST=4 GALA_LIB_PATH=probe_libs/lib_a4b2trace.so B=256 python tools/kf_trace.py > gpurun_out/g9_trace.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "tensor_core or kf or gala2" > gpurun_out/g9_parity.txt 2>&1
cat gpurun_out/g9_probe.txt gpurun_out/g9_trace.txt; tail -3 gpurun_out/g9_parity.txt
