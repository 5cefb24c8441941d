bash tools/gpu_tests.sh tests/test_conv_span_gpu.py tests/test_resnet_gpu.py tests/test_serving_gpu.py tests/test_exchange_gpu.py 2>&1 | grep -E "==|passed|failed|Error|assert" | head -30
python tools/kernel_times.py resnet18 5 2>&1 | grep -v Warn | head -10
