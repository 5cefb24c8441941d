timeout 100 python -m pytest tests/test_gemm_gpu.py tests/test_distilbert_gpu.py -q -x 2>&1 | tail -3
python tools/kernel_times.py distilbert 5 2>&1 | grep -v Warn | sed -n 2,12p
python tools/kernel_times.py distilbert 5 2>&1 | grep -A6 aggregate
