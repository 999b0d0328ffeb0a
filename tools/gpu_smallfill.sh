run() {
  s=$(env "$@" timeout 300 python bench.py --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step']*1e3,1), 'enc', round(d['roofline']['kernel_ms_per_step']['encode']*1e3,1), 'dec', round(d['roofline']['kernel_ms_per_step']['decode']*1e3,1))")
  echo "$* | $s"
}
for rep in 1 2; do
run A8_SCHED_SMALL_MAX=0
run A8_SMALL_KEEP_MAX=1100
run A8_SMALL_KEEP_MAX=1100 A8_SCHED_SMALL_MAX=1100 A8_SCHED_SMALL_FILL=2500
run A8_SMALL_KEEP_MAX=1100 A8_SCHED_SMALL_MAX=1100 A8_SCHED_SMALL_FILL=4000
run A8_SMALL_KEEP_MAX=300 A8_SCHED_SMALL_MAX=300 A8_SCHED_SMALL_FILL=1000
run A8_SMALL_KEEP_MAX=300
done
