# GEMM A/B across libraries built with other compile-time knobs (var/*.so via Q2_LIB_OVERRIDE)
S="16384x11264x2048 16384x2048x11264 16384x2048x2048 2048x5632x16384"
TAG=cur python tools/gemm_one.py $S | grep TF
for v in ${VARS:-}; do Q2_LIB_OVERRIDE=var/$v.so TAG=$v python tools/gemm_one.py $S | grep TF; done
