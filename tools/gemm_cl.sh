# GEMM with clusters of 1, 2, 4 pairs (Q2_GEMM_CL): parity tests + timings, with and without scales
for CL in 1 2 4; do
  echo "== CL=$CL"
  [ -z "${NOTEST:-}" ] && Q2_GEMM_CL=$CL timeout 150 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" 2>&1 | tail -1
  Q2_GEMM_VERBOSE=1 Q2_GEMM_CL=$CL TAG=cl$CL timeout 100 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 2>&1 | grep -E "TF|Error|error|clusters"
  Q2_GEMM_DBG=1 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 Q2_GEMM_CL=$CL TAG=cl${CL}_noscale timeout 100 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 2>&1 | grep -E "TF|Error|error"
done
