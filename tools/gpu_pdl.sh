timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
for pdl in 1 0; do
  A8_PDL=$pdl timeout 300 python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl=$pdl', 'value', round(d['value'],1), 'step', round(d['ms_per_step']*1e3,1), 'enc', round(d['roofline']['kernel_ms_per_step']['encode']*1e3,1), 'dec', round(d['roofline']['kernel_ms_per_step']['decode']*1e3,1))"
done; done
