timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:onebit -s 3 -c 6 --csv python tools/prof_onebit_c3.py 2>/dev/null > gpurun_out/onebit_ncu.csv
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/onebit_ncu.csv")))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[i+1:]:
    print(r[ki][:40], r[mi][:40], r[vi])
PY
