# Grid-barrier encode tuning: C3 bench step per library variant / env (same box, 2 rounds).
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu --no-sweep --steps 20 --warmup 5 > gpurun_out/v.json 2>gpurun_out/v.err || { echo "$name FAILED"; tail -3 gpurun_out/v.err; return; }
  python -c "import json; d=json.loads(open('gpurun_out/v.json').readline()); r=d['roofline']['kernel_ms_per_step']; print('$name', round(d['ms_per_step']*1e3,1), 'enc', round(r['encode']*1e3,1), 'dec', round(r['decode']*1e3,1))"
}
for r in 1 2; do
  run ticket A8_GB=0
  run base
  for v in ${VARS:-r8k4 r12k0 r6k6 r10k2}; do run $v A8_LIB=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; done
  for mb in ${MBS:-0 40 120}; do run L2MB$mb A8_GB_L2MB=$mb; done
done
