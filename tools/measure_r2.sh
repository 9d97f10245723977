set -x
for m in posthoc exact; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_$m.csv python tools/traffic.py run $m > gpurun_out/traffic_run_$m.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
PROF_ENGINE=auto timeout 600 ncu --set full --import-source on --clock-control none -k regex:"msed_tc_kernel|tc_pass2" -c 4 -o gpurun_out/r2_tc_full python tools/prof_tc.py > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:nvfp4_gemm -c 1 -o gpurun_out/r2_gemm_full python tools/gtrace.py > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"quant_fwd|amax" -c 2 -o gpurun_out/r2_quant_full python tools/quant_one.py > /dev/null 2>&1
ls -la gpurun_out
