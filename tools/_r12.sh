timeout 100 python -m pytest tests/test_conv_span_gpu.py tests/test_resnet_gpu.py -q -x 2>&1 | tail -2
for cfg in "GG_SPAN_ASTAGES=2" "GG_SPAN_ASTAGES=3" "GG_SPAN_ASTAGES=4"; do echo "== $cfg"; env $cfg python tools/kernel_times.py resnet18 5 2>&1 | grep -E "span|conv_span" | head -24 | awk '{print $1, $2, $4, $5, $6, $7}'; done
