timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_callers.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/host_overhead_nrank.py; timeout 120 python tools/host_overhead.py
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-sweep --eager 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('eager step', round(r['ms_per_step']*1e3,1))"
