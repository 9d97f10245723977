# SM clock / power / throttle reasons while a GEMM variant runs for a few seconds
run() {
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > /tmp/smi.log &
  P=$!
  env "$@" ITERS=400 timeout 100 python tools/gemm_one.py 16384x2048x11264 2>&1 | grep -E "TF|rror"
  kill $P
  sort /tmp/smi.log | uniq -c | sort -rn | head -4
}
run Q2_GEMM_CL=1 TAG=default
run Q2_GEMM_CL=1 Q2_GEMM_DBG=4 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 TAG=mma_only
run TAG=cublaslt LT=1
