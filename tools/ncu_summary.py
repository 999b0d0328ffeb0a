"""Summarise ncu captures into profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_ncu_summary.txt (per-kernel duration, DRAM bytes,
throughputs, stall mix; launch-list shares) and updates
profiles/ncu_traffic.json with per-launch DRAM bytes keyed "<kernel>_n1"
(read by bench.py as roofline.traffic).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum",
]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, row)), dict(zip(hdr, units))) for row in r[2:]]


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [f"# ncu summary {tag}", f"source: {rep} (--set full --clock-control none), {launches}", ""]
    traffic_path = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for d, u in raw(rep):
        name = "encode" if "encode" in d["Kernel Name"] else "decode" if "decode" in d["Kernel Name"] else d["Kernel Name"]
        lines.append(f"## {d['Kernel Name']}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]} {u.get(k, '')}")
        stalls = sorted(((float(v), k) for k, v in d.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and v not in ("", "n/a")), reverse=True)[:6]
        lines.append("  top stalls (warps per issue): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, k in stalls))
        b = sum(float(d[k]) * UNITS[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        traffic[f"{name}_n1"] = b
        lines.append(f"  dram bytes per launch: {b:.0f}")
        lines.append("")
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, x in enumerate(rows) if x and x[0] == "ID")
    h = rows[hi]
    tot: dict = {}
    for x in rows[hi + 1:]:
        dd = dict(zip(h, x))
        if dd.get("Metric Name") == "gpu__time_duration.sum":
            k = dd["Kernel Name"].split("(")[0]
            tot[k] = tot.get(k, 0.0) + float(dd["Metric Value"])
    s = sum(tot.values())
    lines.append("## launch list shares (cold-cache, serialised: compare shares, not absolutes)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"  {k:50s} {v / 1e3:10.1f} us total  {100 * v / s:5.1f}%")
    out = ROOT / "profiles" / f"{tag}_ncu_summary.txt"
    out.write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print(out.read_text())


if __name__ == "__main__":
    main()
