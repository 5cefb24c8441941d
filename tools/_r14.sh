timeout 100 python -m pytest tests/test_conv_span_gpu.py tests/test_resnet_gpu.py -q -x 2>&1 | tail -4
python tools/kernel_times.py resnet18 5 2>&1 | grep -v Warn | head -30
GG_SPAN_PROF=1 timeout 60 python tools/forward_once.py resnet18 1 2>&1 | grep -E "MMA issuer|^span" | tail -6
