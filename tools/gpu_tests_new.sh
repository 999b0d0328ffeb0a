mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_cli.py tests/test_gpu_onebit.py -m gpu -x -q > gpurun_out/t_new.log 2>&1; echo t_new=$?
tail -15 gpurun_out/t_new.log
timeout 2400 python -m pytest tests/test_dropin_reference.py -m gpu -x -q > gpurun_out/t_dropin.log 2>&1; echo t_dropin=$?
tail -5 gpurun_out/t_dropin.log; tail -5 gpurun_out/dropin_reference_suite.log
