"""Per-phase stall-reason breakdown of an ncu report (source page, SASS view).

    python tools/stall_phases.py <report> <kernel-mangled-name> <lib.so> "name:a-b,name2:file.cuh:c-d" [src-basename]

Phases are line ranges of the kernel source file (default tac_frame.cu); lines
outside every range (headers, intrinsics) are reported as 'other'.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kern, lib, spec = sys.argv[1:5]
srcname = sys.argv[5] if len(sys.argv) > 5 else "tac_frame.cu"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = {}
for f in os.listdir(tmp):
    if not f.endswith(".cubin"):
        continue
    out = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, f)], capture_output=True, text=True).stdout
    if kern not in out:
        continue
    cur_fn, cur_line = None, None
    for ln in out.splitlines():
        if ln.startswith(".text.") or re.match(r"^\s*\.section\s+\.text\.", ln):
            cur_fn = ln.split(".text.")[1].split(",")[0].strip().rstrip(":")
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", ln)
        if m and cur_fn == kern:
            lines_of[int(m.group(1), 16)] = cur_line
    break
phases = []
for s in spec.split(","):
    parts = s.split(":")
    name, rng = parts[0], parts[-1]
    fname = parts[1] if len(parts) == 3 else srcname
    a, b = map(int, rng.split("-"))
    phases.append((name, fname, a, b))
exp = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + os.environ.get("KFILTER", max(re.findall(r"[a-z_]+", kern), key=len))],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(exp)))
hdr = rows[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ii = hdr.index("Instructions Executed")
agg = defaultdict(lambda: defaultdict(float))
k = 0
for r in rows[2:]:
    try:
        v = int(r[ii])
    except (ValueError, IndexError):
        continue
    line = lines_of.get(16 * k)
    k += 1
    ph = "other"
    if line:
        for name, fname, a, b in phases:
            if line[0] == fname and a <= line[1] <= b:
                ph = name
                break
    agg[ph]["instr"] += v
    for c in cols:
        try:
            agg[ph][hdr[c]] += float(r[c] or 0)
        except ValueError:
            pass
tot = sum(sum(v for kk, v in d.items() if kk != "instr") for d in agg.values())
for ph, d in agg.items():
    s = sum(v for kk, v in d.items() if kk != "instr")
    top = sorted(((v, kk) for kk, v in d.items() if kk != "instr"), reverse=True)[:6]
    print(f"{ph:10s} samples {100 * s / tot:5.1f}%  instr {d['instr']:.3g}  " +
          " ".join(f"{kk[6:]}={100 * v / tot:.1f}" for v, kk in top))
