# Same-box A/B of several _lib_var builds against the product build (bench encode/decode times).
mkdir -p gpurun_out
: > gpurun_out/ab_multi.txt
for rep in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  A8_LIB=$lib timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']
    print('$v', 'step', round(r['ms_per_step']*1e3,1), 'enc', round(k['encode']*1e3,1), 'dec', round(k['decode']*1e3,1))" | tee -a gpurun_out/ab_multi.txt
done; done
