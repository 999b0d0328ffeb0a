A8_LIB=paper_1511_04561_b200/_lib_var/bld/libapprox8_b200.so timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_segments.py -m gpu -x -q 2>&1 | tail -2
for wf in 1200 2500 4000 6432; do
for v in base bld; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  if [ $v = base ] && [ $wf != 6432 ]; then continue; fi
  A8_SCHED_FILL=$wf A8_LIB=$lib timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']
    print('$v wf=$wf', 'step', round(r['ms_per_step']*1e3,1), 'enc', round(k['encode']*1e3,1), 'dec', round(k['decode']*1e3,1))"
done; done
