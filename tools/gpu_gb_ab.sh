# Grid-barrier encode vs the ticket kernel (A8_GB=0) on the C3 bench step, same box; tuning builds in _lib_var/.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large_calls.py tests/test_gpu_fuzz.py tests/test_gpu_bench_step.py -x -q 2>&1 | tail -2
run() { local name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --warmup 5 > gpurun_out/v.json 2>gpurun_out/v.err || { echo "$name FAILED"; tail -3 gpurun_out/v.err; return; }
  python -c "import json; d=json.loads(open('gpurun_out/v.json').readline()); r=d['roofline']['kernel_ms_per_step']; print('$name', round(d['ms_per_step']*1e3,1), 'enc', round(r['encode']*1e3,1), 'dec', round(r['decode']*1e3,1))"; }
L=paper_1511_04561_b200/_lib_var
for r in 1 2; do
  run ticket A8_GB=0; run gb80; run gb40 A8_GB_L2MB=40; run gb120 A8_GB_L2MB=120
  run nodem80 A8_LIB=$L/nodem/libapprox8_b200.so
done
