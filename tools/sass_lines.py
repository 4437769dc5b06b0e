"""Attribute ncu per-instruction SASS metrics to CUDA source lines.

    python tools/sass_lines.py <report.ncu-rep> <kernel-mangled-name> [lib.so]

Uses `nvdisasm -g` line tables of the kernel's cubin (built with -lineinfo)
and the `--page source --print-source sass` export of the report; the k-th
SASS row of the export is the instruction at offset 16*k of the function.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2411_04776_b200/libtac_b200.so"

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
            name = ln.split(".text.")[1].split(",")[0].strip().rstrip(":")
            cur_fn = name
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", ln)
        if m and cur_fn == kern:
            lines_of[int(m.group(1), 16)] = (cur_line, m.group(2))
    break

exp = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + os.environ.get("KFILTER", max(re.findall(r"[a-z_]+", kern), key=len))],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(exp)))
hdr = rows[1]
ii = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
k = 0
for r in rows[2:]:
    try:
        v, s = int(r[ii]), int(r[si])
    except (ValueError, IndexError):
        continue
    line = lines_of.get(16 * k, (None, ""))[0]
    agg[line][0] += v
    agg[line][1] += s
    tot_i += v
    tot_s += s
    k += 1
print(f"{k} sass rows, {len(lines_of)} mapped offsets, total instr {tot_i}")
for line, (v, s) in sorted(agg.items(), key=lambda t: -t[1][1])[:40]:
    print(f"{str(line):40s} instr {100 * v / tot_i:5.1f}%  stall {100 * s / tot_s:5.1f}%")

if len(sys.argv) > 4:
    # optional: phase ranges "name:a-b,name2:c-d" over tac_frame.cu lines
    ph = defaultdict(lambda: [0, 0])
    for spec in sys.argv[4].split(","):
        name, rng = spec.split(":")
        a, b = map(int, rng.split("-"))
        for line, (v, s) in agg.items():
            if line and line[0] == "tac_frame.cu" and a <= line[1] <= b:
                ph[name][0] += v
                ph[name][1] += s
    for name, (v, s) in ph.items():
        print(f"PHASE {name:12s} instr {100 * v / tot_i:5.1f}%  ({v * 32 / float(os.environ.get('PIXELS', 1)):.1f}/px)  stall {100 * s / tot_s:5.1f}%")

if os.environ.get("LINES"):
    a, b = map(int, os.environ["LINES"].split("-"))
    srcf = os.environ.get("SRC", "paper_2411_04776_b200/csrc/tac_frame.cu")
    src = open(srcf).read().splitlines()
    px = float(os.environ.get("PIXELS", 1))
    for line, (v, s) in sorted((k, t) for k, t in agg.items() if k and k[0] == os.path.basename(srcf)):
        if a <= line[1] <= b and v:
            print(f"L{line[1]:5d} {v * 32 / px:6.2f}/px stall {100 * s / tot_s:5.1f}%  {src[line[1] - 1].strip()[:90]}")
