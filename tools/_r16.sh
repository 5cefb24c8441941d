timeout 100 python -m pytest tests/test_conv_span_gpu.py tests/test_resnet_gpu.py tests/test_serving_gpu.py -q -x 2>&1 | tail -4
python tools/kernel_times.py resnet18 5 2>&1 | grep -v Warn | head -30
