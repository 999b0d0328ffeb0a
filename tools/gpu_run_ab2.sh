V=${1:-pf}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_ab_enc.sh $V
for wf in 3000 4500 6432; do echo "wf=$wf"; A8_SCHED_FILL=$wf A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so timeout 300 python tools/switch_trace.py 2>&1 | tail -4; A8_SCHED_FILL=$wf timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']; print('enc', round(k['encode']*1e3,1))"; done
