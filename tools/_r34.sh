bash tools/gpu_tests.sh tests/test_distilbert_gpu.py tests/test_serving_gpu.py tests/test_gemm_gpu.py 2>&1 | grep -E "==|passed|failed|Error|assert" | head -30
python tools/kernel_times.py distilbert 5 2>&1 | grep -v Warn | sed -n 2,9p
python tools/kernel_times.py distilbert 5 2>&1 | grep -A6 aggregate
