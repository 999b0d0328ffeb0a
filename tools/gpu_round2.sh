# Round run: smoke, all GPU tests, bench (both arms), launch list and ncu captures.
set -x
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref=$?
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep > /dev/null 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel|decode_kernel|decode_tma_kernel" -s 6 -c 2 -o gpurun_out/full python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep > gpurun_out/ncu_full.log 2>&1; echo full=$?
