timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_callers.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for t in 0 1; do
A8_DEC_TMA=$t timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']
    print('tma=$t', 'step', round(r['ms_per_step']*1e3,1), 'enc', round(k['encode']*1e3,1), 'dec', round(k['decode']*1e3,1))"
done; done
A8_DEC_TMA=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed -k regex:decode -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep 2>/dev/null | tail -4
