run() {
  s=$(timeout 300 python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step']*1e3,1), 'enc', round(d['roofline']['kernel_ms_per_step']['encode']*1e3,1), 'dec', round(d['roofline']['kernel_ms_per_step']['decode']*1e3,1))")
  e=$(timeout 300 python tools/prof_codec.py --case big --iters 5 2>&1 | grep 2^30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2^30 enc', round(d['encode']['ms']*1e3,1))")
  echo "$1 | $s | $e"
}
for rep in 1 2; do
  unset A8_LIB; run product
  for v in b1 b4 s3 s5; do export A8_LIB=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; run $v; done
done
