# Same-box A/B of the product build against paper_1511_04561_b200/_lib_var/head (the last commit).
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
A8_RESIDENT=0 timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_codec.py -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/pt.txt
for rep in 1 2; do
for v in base head; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  for c in alexnet mlpcodec; do A8_LIB=$lib A8_RESIDENT=0 timeout 300 python tools/prof_codec.py --case $c | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', r['case'], 'enc', round(r['encode']['ms']*1e3,1))"; done
  A8_LIB=$lib python tools/prof_roundtrip.py > gpurun_out/rt_$v.txt 2>&1; head -2 gpurun_out/rt_$v.txt | sed "s/^/$v /"
done
done
cat gpurun_out/pt.txt
