# Encode schedule knobs at C3: A8_SCHED_FILL (fill distance in tickets) x A8_CODE_HINT,
# event time from bench.py and DRAM read/write bytes from ncu (separate runs).
mkdir -p gpurun_out
: > gpurun_out/sched_sweep.txt
for hint in 0 1; do
for wf in 1200 2000 3000 4500 6432; do
  t=$(A8_CODE_HINT=$hint A8_SCHED_FILL=$wf timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-sweep 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); k=r['roofline']['kernel_ms_per_step']; print(round(k['encode']*1e3,1), round(k['decode']*1e3,1), round(r['ms_per_step']*1e3,1))")
  b=$(A8_CODE_HINT=$hint A8_SCHED_FILL=$wf timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:encode_kernel -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep 2>/dev/null | grep -E "dram__bytes|hit_rate" | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | paste -sd' ')
  echo "hint=$hint wf=$wf enc/dec/step_us=$t $b" | tee -a gpurun_out/sched_sweep.txt
done
done
