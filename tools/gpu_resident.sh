mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log; done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_errorbench.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -1; done
A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so python tools/res_trace.py
for r in 1 0; do
  A8_RESIDENT=$r timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/res_$r.csv python tools/prof_codec.py --case mlpcodec --iters 3 > /dev/null 2>&1; echo rc=$?
done
