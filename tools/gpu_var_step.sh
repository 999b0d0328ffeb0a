# Same-box A/B of tuning builds (paper_1511_04561_b200/_lib_var/<name>) on the C3 bench step, 2 rounds.
# usage: VARS="name1 name2" bash tools/gpu_var_step.sh
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --warmup 5 > gpurun_out/v.json 2>gpurun_out/v.err || { echo "$name FAILED"; tail -3 gpurun_out/v.err; return; }
  python -c "import json; d=json.loads(open('gpurun_out/v.json').readline()); r=d['roofline']['kernel_ms_per_step']; print('$name', round(d['ms_per_step']*1e3,1), 'enc', round(r['encode']*1e3,1), 'dec', round(r['decode']*1e3,1))"
}
for r in 1 2; do
  run base
  for v in $VARS; do run $v A8_LIB=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; done
done
