"""Summarise an ncu --set full report (one section per captured kernel) into profiles/.

    python tools/ncu_summary.py <report.ncu-rep> <out.md> [--traffic-key configs[2] --envs N]

With --traffic-key, writes DRAM read+write bytes per launch of every kernel
(and the env count of the captured launch) into profiles/traffic.json, which
bench.py reads for roofline.traffic.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
args = sys.argv[3:]
key = args[args.index("--traffic-key") + 1] if "--traffic-key" in args else None
envs = int(args[args.index("--envs") + 1]) if "--envs" in args else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = [
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def mb(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


lines, traffic = [], {}
for vals in rows[2:]:
    d = {n: (vals[i], units[i]) for i, n in enumerate(h)}
    name = d["Kernel Name"][0]
    m = re.search(r"(\w+_kernel)(<(\w+)[,>])?", name)
    short = m.group(1) if m else name
    if short == "band_shade_kernel" and m.group(3) in ("true", "1"):
        short = "band_shade_kernel<f16 LUT>"
    if short == "shadow_tiled_kernel":
        short = "shadow_kernel"  # bench.py's name for the march
    lines += [f"## {name}", "", "| metric | value |", "|---|---|"]
    for k, label in want:
        if k in d:
            v, u = d[k]
            lines.append(f"| {label} (`{k}`) | {v} {u} |")
    stalls = []
    for n, (v, u) in d.items():
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    lines.append("")
    lines.append("Top warp-stall reasons (warps stalled per issued instruction): " +
                 ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
    t = mb(*d["dram__bytes_read.sum"]) + mb(*d["dram__bytes_write.sum"])
    traffic[short] = traffic.get(short, t)
    lines += [f"\nDRAM traffic per launch: {t:.0f} B", ""]
with open(out, "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
if key:
    tpath = os.path.join(os.path.dirname(out), "traffic.json")
    doc = json.load(open(tpath)) if os.path.exists(tpath) else {}
    entry = dict(traffic)
    if envs:
        entry["envs"] = envs
    doc.setdefault(key, {}).update(entry)
    json.dump(doc, open(tpath, "w"), indent=1)
