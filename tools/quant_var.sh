# forward quantizer A/B: libraries built with other register caps (var/*.so via Q2_LIB_OVERRIDE)
TAG=cur python tools/quant_probe.py | grep total
for v in ${VARS:-}; do echo "== $v"; Q2_LIB_OVERRIDE=var/$v.so python tools/quant_probe.py | grep total; done
