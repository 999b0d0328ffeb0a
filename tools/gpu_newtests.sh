timeout 900 python -m pytest tests/test_gpu_premax.py tests/test_gpu_bench_step.py -q 2>&1 | tail -4
