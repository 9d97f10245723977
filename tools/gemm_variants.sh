S="16384x11264x2048 16384x2048x11264"
TAG=default python tools/gemm_one.py $S
TAG=mask0 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 python tools/gemm_one.py $S
TAG=mask1F Q2_GEMM_CPMASK_SHORT=0x1F Q2_GEMM_CPMASK_LONG=0x1F python tools/gemm_one.py $S
TAG=mask0_dbg1 Q2_GEMM_DBG=1 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 python tools/gemm_one.py $S
TAG=cp Q2_GEMM_CP=1 python tools/gemm_one.py $S
