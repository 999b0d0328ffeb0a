mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_onebit.py tests/test_gpu_codec.py tests/test_f64.py tests/test_tensorfile.py tests/test_errorbench.py -m gpu -x -q > gpurun_out/t1.log 2>&1; echo t1=$?
tail -30 gpurun_out/t1.log
timeout 1800 python -m pytest tests/test_dropin_reference.py -m gpu -x -q > gpurun_out/t2.log 2>&1; echo t2=$?
tail -30 gpurun_out/t2.log
tail -30 gpurun_out/dropin_reference_suite.log
