python tools/prof_onebit_c3.py
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -s 100 -c 60 --csv python tools/prof_onebit_c3.py 2>/dev/null > gpurun_out/onebit_ncu.csv
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/onebit_ncu.csv")))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i]; ki, mi, vi, gi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Grid Size") if "Grid Size" in h else None
for r in rows[i+1:]:
    print(r[ki][:40], r[mi][:40], r[vi], r[gi] if gi else "")
PY
