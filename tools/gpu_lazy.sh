timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
A8_RESIDENT=0 timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_codec.py tests/test_gpu_exchange.py -m gpu -x -q 2>&1 | tail -1
for v in base head; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  A8_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lazy_$v.csv python tools/prof_codec.py --case alexnet --iters 3 > /dev/null 2>&1
  for c in alexnet big; do A8_LIB=$lib A8_RESIDENT=0 timeout 300 python tools/prof_codec.py --case $c | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', r['case'], 'enc', round(r['encode']['ms']*1e3,1), 'us dec', round(r['decode']['ms']*1e3,1))"; done
done
A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so timeout 300 python tools/ticket_trace.py --case alexnet --out gpurun_out/tt_lazy.json > gpurun_out/tt_lazy.txt 2>&1
