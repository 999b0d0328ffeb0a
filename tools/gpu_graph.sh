mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_callers.py -m gpu -x -q > gpurun_out/pytest_graph.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_graph.log
for st in 20 100; do
timeout 600 python bench.py --no-cpu --steps $st > gpurun_out/bench_g.json; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_g.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step'])"
done
