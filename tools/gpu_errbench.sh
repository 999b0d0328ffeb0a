mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_errorbench.py -m gpu -x -q > gpurun_out/pytest_err.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_err.log
timeout 600 python tools/errorbench_timing.py > gpurun_out/errorbench_timing.jsonl 2>&1; echo timing=$?
cat gpurun_out/errorbench_timing.jsonl | head -3
grep suite_gpu gpurun_out/errorbench_timing.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:error_stats -s 2 -c 1 -o gpurun_out/errstats python tools/errorbench_timing.py --cpu-n 1000 > /dev/null 2>&1; echo ncu=$?
