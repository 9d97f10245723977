# ncu: our GEMM (normal, MMA-only probe) vs the cuBLASLt NVFP4 kernel at the dgrad shape
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_active"
S=16384x2048x11264
Q2_GEMM_CL=1 ITERS=2 ncu --clock-control none --metrics $M -k regex:nvfp4_gemm -c 2 --csv python tools/gemm_one.py $S > gpurun_out/ncu_ours.csv 2>&1
Q2_GEMM_CL=1 Q2_GEMM_DBG=4 Q2_GEMM_CPMASK_SHORT=0 Q2_GEMM_CPMASK_LONG=0 ITERS=2 ncu --clock-control none --metrics $M -k regex:nvfp4_gemm -c 2 --csv python tools/gemm_one.py $S > gpurun_out/ncu_mmaonly.csv 2>&1
LT=1 ITERS=2 ncu --clock-control none --metrics $M -k regex:cutlass -c 2 --csv python tools/gemm_one.py $S > gpurun_out/ncu_lt.csv 2>&1
for f in ours mmaonly lt; do echo "== $f"; grep -E '^"[0-9]' gpurun_out/ncu_$f.csv | awk -F'","' '{print $(NF-3), $(NF-2), $NF}' | tail -8; done
