for v in base bl6 bl8; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  A8_LIB=$lib python tools/prof_blocked.py | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if r['log2'] in (26,30): print('$v', r['log2'], r['block'], round(r['encode_us'],1), round(r['encode_GBps']))"
done
