# tensor-pipe rate probes (wrong results): 4 = MMAs re-read the first stages, 5 = same with
# kind::mxf4 block32, 6 = kind::f8f6f4 (E2M1, no scales, K=32 per instruction)
for D in 4 7 4 7; do
  Q2_GEMM_CL=1 Q2_GEMM_DBG=$D Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 TAG=dbg$D timeout 60 python tools/gemm_one.py 16384x2048x11264 2>&1 | grep -E "TF|rror"
done
