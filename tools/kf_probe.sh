# k_gala_kf role isolation and ring depths (experiment builds; the probe flags give garbage words):
#   sh tools/kf_probe.sh build   (here: one library per variant into probe_libs/)
#   sh tools/kf_probe.sh         (on the box: tools/time_fc.py against each)
NAMES=${NAMES:-"base onlyMMA noA noB noE"}
flags() {
  case $1 in
    base) echo "" ;; noA) echo "-DKF_NO_A" ;; noW) echo "-DKF_NO_W" ;; noB) echo "-DKF_NO_B" ;; noE) echo "-DKF_NO_EPI" ;;
    onlyMMA) echo "-DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;; noAnoB) echo "-DKF_NO_A -DKF_NO_B" ;;
    j8s3) echo "-DKF_JS=8 -DKF_ST=3" ;; j8s3w32) echo "-DKF_JS=8 -DKF_ST=3 -DKF_WJ=32 -DKF_WST=2" ;;
    j8s3trace) echo "-DKF_JS=8 -DKF_ST=3 -DKF_TRACE" ;; j8s3only) echo "-DKF_JS=8 -DKF_ST=3 -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    j8s3noA) echo "-DKF_JS=8 -DKF_ST=3 -DKF_NO_A" ;; j8s3noB) echo "-DKF_JS=8 -DKF_ST=3 -DKF_NO_B" ;; j8s3noE) echo "-DKF_JS=8 -DKF_ST=3 -DKF_NO_EPI" ;;
    a4b2) echo "" ;; a3b3) echo "-DKF_AST=3 -DKF_BST=3" ;; a5b1) echo "-DKF_AST=5 -DKF_BST=1" ;;
    j4a8b4) echo "-DKF_JS=4 -DKF_AST=8 -DKF_BST=4" ;; j4a10b2) echo "-DKF_JS=4 -DKF_AST=10 -DKF_BST=2" ;;
    a4b2only) echo "-DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;; a4b2trace) echo "-DKF_TRACE" ;;
    wsplit) echo "-DKF_WSPLIT" ;; wsplit_a4) echo "-DKF_WSPLIT -DKF_JS=8 -DKF_ST=3 -DKF_WST=4" ;; wsplit_w32) echo "-DKF_WSPLIT -DKF_WJ=32 -DKF_WST=2" ;;
    st4w2) echo "-DKF_ST=4 -DKF_WJ=8 -DKF_WST=2" ;; js16st1) echo "-DKF_JS=16 -DKF_ST=1 -DKF_WJ=16 -DKF_WST=4" ;;
    flag) echo "" ;; flagvol) echo "-DKF_FLAG_VOLATILE" ;; noflag) echo "-DKF_NO_FLAG" ;;
    flagonly) echo "-DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;; flagtrace) echo "-DKF_TRACE" ;;
    flagonlytrace) echo "-DKF_TRACE -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;; noflagonlytrace) echo "-DKF_NO_FLAG -DKF_TRACE -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    j16s1) echo "-DKF_JS=16 -DKF_ST=1" ;; j8s2w32) echo "-DKF_JS=8 -DKF_ST=2 -DKF_WJ=32 -DKF_WST=2" ;;
    j4s4) echo "-DKF_JS=4 -DKF_ST=4" ;; j8s2) echo "-DKF_JS=8 -DKF_ST=2" ;;
    j4s4_onlyMMA) echo "-DKF_JS=4 -DKF_ST=4 -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    j8s2_onlyMMA) echo "-DKF_JS=8 -DKF_ST=2 -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    j4s4_noB) echo "-DKF_JS=4 -DKF_ST=4 -DKF_NO_B" ;;
    susp) echo "-DKF_SUSPEND=1000000" ;; susp_onlyMMA) echo "-DKF_SUSPEND=1000000 -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    trace_susp_onlyMMA) echo "-DKF_TRACE -DKF_SUSPEND=1000000 -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
    trace) echo "-DKF_TRACE" ;; trace1) echo "-DKF_TRACE -DKF_TRACE_CTA=1" ;; trace_onlyMMA) echo "-DKF_TRACE -DKF_NO_A -DKF_NO_W -DKF_NO_B -DKF_NO_EPI" ;;
  esac
}
if [ "$1" = "build" ]; then
  mkdir -p probe_libs
  for n in $NAMES; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $(flags $n) \
      -o probe_libs/lib_$n.so paper_2105_01827_b200/csrc/gala_lib.cu -L/usr/local/cuda/lib64 -Xlinker -rpath=/usr/local/cuda/lib64 2>/dev/null &
  done
  wait
else
  for n in $NAMES; do
    echo "$n: $(GALA_LIB_PATH=probe_libs/lib_$n.so B=${B:-128} python tools/time_fc.py 2>&1 | tail -1 | cut -c1-60)"
  done
fi
