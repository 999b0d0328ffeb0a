# A/B of tuning builds (paper_1511_04561_b200/_lib_var/<name>) against the product library.
# usage: bash tools/ab_variants.sh name1 name2 ...
mkdir -p gpurun_out
out=gpurun_out/ab_variants.jsonl; : > $out
for v in base "$@"; do
  if [ "$v" = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  A8_LIB=$lib python -c "
import ctypes as C, json
from paper_1511_04561_b200 import _native as N
a,b,c=C.c_int(),C.c_int(),C.c_int(); N.lib.a8_device_info(0,C.byref(a),C.byref(b),C.byref(c)); print(json.dumps({'variant':'$v','sms':a.value,'enc_occ':b.value,'dec_occ':c.value}))" >> $out
  for spec in dynamic-tree/absmax mantissa/decade+1; do
    for case in alexnet big; do
      A8_LIB=$lib timeout 300 python tools/prof_codec.py --case $case --spec $spec | sed "s/^/{\"variant\":\"$v\",\"r\":/; s/$/}/" >> $out
    done
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/ab_variants.jsonl'):
    d=json.loads(l)
    if 'r' not in d: print(d); continue
    r=d['r']; print(f"{d['variant']:8s} {r['case']:12s} {r['spec']:22s} enc {r['encode']['ms']*1e3:8.1f} us  dec {r['decode']['ms']*1e3:8.1f} us")
PY
