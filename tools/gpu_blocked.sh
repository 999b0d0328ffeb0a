mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_blocked.py tests/test_gpu_onebit.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/prof_blocked.py 2>&1 | tail -14
timeout 600 ncu --set full --clock-control none -k regex:"blocked_encode_stream" -s 2 -c 1 -o gpurun_out/full_blocked python tools/prof_blocked.py > /dev/null 2>&1; echo ncu=$?
