# MS-EDEN A/B on one box: current build vs var/*.so (Q2_LIB_OVERRIDE), c3 UpGate and Down shapes
for v in cur ${VARS:-}; do
  if [ "$v" = cur ]; then L=""; else L=var/$v.so; fi
  for rep in 1 2; do
    Q2_LIB_OVERRIDE=$L timeout 120 python tools/tc_probe.py 2>&1 | grep dbg | sed "s/^/[$v] /"
  done
  Q2_LIB_OVERRIDE=$L IN=5632 OUT=2048 timeout 120 python tools/tc_probe.py 2>&1 | grep posthoc | sed "s/^/[$v] /"
done
