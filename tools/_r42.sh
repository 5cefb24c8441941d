bash tools/gpu_tests.sh tests/test_resnet_gpu.py 2>&1 | grep -E "==|passed|failed|Error|assert" | head
python tools/kernel_times.py resnet18 5 2>&1 | grep -v Warn | head -6
python tools/kernel_times.py resnet18 5 2>&1 | grep "forward span"
