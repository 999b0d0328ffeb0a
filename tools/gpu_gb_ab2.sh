mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gbencode.py tests/test_gpu_bench_step.py -x -q > gpurun_out/gb_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gb_tests.log
A8_LIB=paper_1511_04561_b200/_lib_var/tr/libapprox8_b200.so timeout 300 python tools/gb_trace.py
VARS="" MBS="0 40" bash tools/gpu_gb_var.sh
