# does the operand data change the GEMM rate (power)?  random vs all-zero codes, ours and cuBLASLt
S=16384x2048x11264
for Z in "" 1; do
  ZERO=$Z Q2_GEMM_CL=1 TAG=ours_zero$Z python tools/gemm_one.py $S 2>&1 | grep TF
  ZERO=$Z Q2_GEMM_CL=1 Q2_GEMM_DBG=4 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 TAG=mma_only_zero$Z python tools/gemm_one.py $S 2>&1 | grep TF
  ZERO=$Z LT=1 TAG=lt_zero$Z python tools/gemm_one.py $S 2>&1 | grep TF
done
