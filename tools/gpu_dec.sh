A8_RESIDENT=0 timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_codec.py tests/test_gpu_exchange.py -m gpu -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do
for v in base head; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  for spec in dynamic-tree/absmax mantissa/decade+1; do
  for c in alexnet big; do A8_LIB=$lib A8_RESIDENT=0 timeout 300 python tools/prof_codec.py --case $c --spec $spec | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', r['spec'][:8], r['case'], 'enc', round(r['encode']['ms']*1e3,1), 'us dec', round(r['decode']['ms']*1e3,1))"; done
  done
done
done
A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so timeout 300 python tools/ticket_trace.py --case alexnet --out gpurun_out/tt_now.json > gpurun_out/tt_now.txt 2>&1
