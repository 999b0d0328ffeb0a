"""Per-region instruction / stall-sample shares of one kernel in an ncu report
(source page, SASS): python tools/ncu_src_regions.py REPORT KERNEL_REGEX"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, sa = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > 10 and r[ia].isdigit()]
tot = sum(int(r[ia]) for r in data)
stot = sum(int(r[sa]) for r in data) or 1
print("warp instructions", tot, "stall samples", stot)
top = sorted(range(len(data)), key=lambda i: -int(data[i][sa]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]
for i in sorted(top):
    r = data[i]
    print(f"{i:6d} {r[1][:70]:70s} {r[ia]:>10s} {int(r[sa]) / stot * 100:5.1f}%")
