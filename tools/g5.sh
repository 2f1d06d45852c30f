mkdir -p gpurun_out
GALA_LIB_PATH=probe_libs/lib_trace.so B=256 python tools/kf_trace.py > gpurun_out/g5_trace.txt 2>&1
RANK1=1 GALA_LIB_PATH=probe_libs/lib_trace1.so B=256 python tools/kf_trace.py > gpurun_out/g5_trace1.txt 2>&1
echo done
