mkdir -p gpurun_out
A8_ENC_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for sp in 0 1; do
A8_ENC_SPLIT=$sp timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']
    print('split=$sp', 'step', round(r['ms_per_step']*1e3,1), 'enc', round(k['encode']*1e3,1), 'dec', round(k['decode']*1e3,1), 'frac', round(r['roofline']['frac'],3))"
done; done
A8_ENC_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:encode_kernel -s 6 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep 2>/dev/null | grep -E "encode" | awk -F'","' '{print $(NF-2)"="$NF}'
