run() {
  r=$(env "$@" timeout 300 python tools/prof_codec.py --case alexnet 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['encode']['ms']*1e3,1))")
  s=$(env "$@" timeout 300 python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step']*1e3,1), 'enc', round(d['roofline']['kernel_ms_per_step']['encode']*1e3,1), 'dec', round(d['roofline']['kernel_ms_per_step']['decode']*1e3,1))")
  echo "$* encode_us=$r | $s"
}
export A8_POL_A=0 A8_POL_E=0
for rep in 1 2; do
run A8_CODE_HINT=0
run A8_CODE_HINT=1
run A8_CODE_HINT=2
run A8_SCHED_FILL=2000
run A8_SCHED_FILL=4000
run A8_SCHED_FILL=9000
run A8_SCHED_POOL=1
done
