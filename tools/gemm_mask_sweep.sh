# scale-path split sweep: copier mask (stages whose scales go by tcgen05.cp) and MMA-thread cp
S="16384x11264x2048 16384x2048x11264 2048x5632x16384"
for M in 0x00 0x15 0x1F 0x0A 0x1B; do
  Q2_GEMM_CPMASK_SHORT=$M Q2_GEMM_CPMASK_LONG=$M TAG=mask$M timeout 60 python tools/gemm_one.py $S 2>&1 | grep -E "TF|rror"
done
Q2_GEMM_CP=1 TAG=mma_cp timeout 60 python tools/gemm_one.py $S 2>&1 | grep -E "TF|rror"
