timeout 900 ncu --set full --clock-control none -k regex:blocked_encode_stream -s 2 -c 1 -o gpurun_out/blk python tools/prof_blocked_one.py 28 4096 3 > /dev/null 2>&1; echo rc=$?
ncu -i gpurun_out/blk.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
want=['gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum']
for w in want:
    if w in h: print(w, v[h.index(w)])
st=[(h[i], v[i]) for i in range(len(h)) if h[i].startswith('smsp__average_warp_latency_issue_stalled') or h[i].startswith('smsp__average_warps_issue_stalled_')]
def f(x):
    try: return float(x)
    except: return 0
st=sorted(st,key=lambda t:-f(t[1]))[:8]
for a,b in st: print(a,b)
"
