# ncu L2 throughput / duration / clock: clusters of 1 vs 2 pairs (dgrad shape)
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum"
S=16384x2048x11264
for CL in 1 2; do
  Q2_GEMM_CL=$CL ITERS=2 WARM=1 ncu --clock-control none --metrics $M -k regex:nvfp4_gemm -c 2 --csv python tools/gemm_one.py $S > gpurun_out/ncu_cl$CL.csv 2>&1
done
LT=1 ITERS=2 WARM=1 ncu --clock-control none --metrics $M -k regex:cutlass -c 2 --csv python tools/gemm_one.py $S > gpurun_out/ncu_lt2.csv 2>&1
for f in cl1 cl2 lt2; do echo "== $f"; grep -E '^"[0-9]' gpurun_out/ncu_$f.csv | awk -F'","' '{print $(NF-3), $(NF-2), $NF}' | tail -7; done
