# GEMM parity tests + c3 timings (+ MMA-only probe) for the current build
timeout 150 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" 2>&1 | tail -1
Q2_GEMM_CL=${CL:-1} TAG=cur timeout 100 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 16384x2048x2048 16384x5632x2048 2048x5632x16384 2>&1 | grep -E "TF|rror"
Q2_GEMM_CL=1 Q2_GEMM_DBG=4 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 TAG=mma_only timeout 60 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 2>&1 | grep -E "TF|rror"
LT=1 TAG=cublaslt timeout 60 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 2>&1 | grep -E "TF|rror"
Q2_GEMM_CL=1 Q2_GEMM_DBG=1 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 TAG=noscale timeout 60 python tools/gemm_one.py 16384x11264x2048 16384x2048x11264 2>&1 | grep -E "TF|rror"
