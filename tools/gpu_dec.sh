timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
for v in base head; do
  if [ $v = base ]; then lib=$PWD/paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=$PWD/paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  (cd tools && A8_LIB=$lib python prof_decode_reduce.py | sed "s/^/$v /")
  for c in alexnet big; do A8_LIB=$lib timeout 300 python tools/prof_codec.py --case $c | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', r['case'], 'enc', round(r['encode']['ms']*1e3,1), 'us dec', round(r['decode']['ms']*1e3,1))"; done
done
