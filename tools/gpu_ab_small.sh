# Same-box A/B of small-call latency: product build vs paper_1511_04561_b200/_lib_var/$1.
V=${1:-head}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
for rep in 1 2; do
for v in base $V; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  for c in small mlpcodec; do A8_LIB=$lib timeout 300 python tools/prof_codec.py --case $c | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', r['case'], 'enc', round(r['encode']['ms']*1e3,1), 'dec', round(r['decode']['ms']*1e3,1))"; done
  A8_LIB=$lib python tools/prof_roundtrip.py 2>&1 | sed "s/^/$v /"
done
done
cat gpurun_out/pt.txt
