NAMES="j8s3 j8s3only j8s3noA j8s3noB j8s3noE" B=256 sh tools/kf_probe.sh > gpurun_out/g8_probe.txt 2>&1
NST=8 ST=3 GALA_LIB_PATH=probe_libs/lib_j8s3trace.so B=256 python tools/kf_trace.py > gpurun_out/g8_trace.txt 2>&1
cat gpurun_out/g8_probe.txt gpurun_out/g8_trace.txt
