# Same-box A/B of bench.py: the product build against paper_1511_04561_b200/_lib_var/$1.
V=${1:-head}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
for rep in 1 2 3; do
for v in base $V; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  A8_LIB=$lib timeout 300 python bench.py --steps 200 --warmup 5 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$v', round(r['value'],1), round(r['ms_per_step']*1e3,1), 'us', 'e2e', round(r['e2e']['value'],2))" >> gpurun_out/ab_bench.txt
done
done
cat gpurun_out/pt.txt gpurun_out/ab_bench.txt
