# Grid-barrier encode: parity tests, then same-box A/B of the C3 bench step (A8_GB=0: ticket kernel).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gbencode.py -x -q > gpurun_out/gb_tests.log 2>&1; echo gbtests=$?
tail -15 gpurun_out/gb_tests.log
timeout 900 python -m pytest tests/test_gpu_bench_step.py tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_segments.py -x -q > gpurun_out/gb_tests2.log 2>&1; echo tests2=$?
tail -3 gpurun_out/gb_tests2.log
for r in 1 2; do
  for v in 0 1; do
    A8_GB=$v timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --warmup 5 > gpurun_out/gb_ab_$v_$r.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/gb_ab_$v_$r.json').readline()); print('GB=$v', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['roofline']['kernel_ms_per_step'], d['roofline']['frac'])"
  done
done
