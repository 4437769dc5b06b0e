"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py <launches.csv> <out.txt> "<command line>"
"""
import csv
import sys
from collections import defaultdict

src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [l for l in open(src) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        agg[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
out_lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none ({cmd})",
             "launches  mean_us  share_of_listed_time  kernel"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    out_lines.append(f"{len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / tot:6.1f}%  {k[:90]}")
ours = {k: v for k, v in agg.items() if "tac::" in k}
t_ours = sum(sum(v) for v in ours.values())
out_lines.append("")
out_lines.append("share of this repo's kernels within the tac_pipeline launches:")
for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
    out_lines.append(f"  {100 * sum(v) / t_ours:5.1f}%  {k[:90]}")
open(out, "w").write("\n".join(out_lines) + "\n")
print("\n".join(out_lines))
