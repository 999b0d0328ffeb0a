timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
for v in base head; do
  if [ $v = base ]; then lib=$PWD/paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=$PWD/paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  (cd tools && A8_LIB=$lib python prof_decode_reduce.py | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v N', r['nranks'], round(r['decode_reduce_us'],1))")
  A8_LIB=$lib python tools/sweep_config4.py --max-log2 22 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if r['spec']=='dynamic-tree/absmax': print('$v', r['log2'], 'dec', round(r['decode_us'],1))"
done
cat gpurun_out/pt.txt
