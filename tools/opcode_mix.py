"""Dynamic SASS opcode mix of one kernel in an ncu report (source page).

    python tools/opcode_mix.py <report> <kernel-substring> [pixels]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
px = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
mix = Counter()
tot = 0
for r in rows[2:]:
    try:
        n = int(r[ii])
    except (ValueError, IndexError):
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)", r[si])
    op = m.group(2).split(".")[0] if m else "?"
    mix[op] += n
    tot += n
for op, n in mix.most_common(30):
    extra = f"  {n * 32 / px:6.2f}/px" if px else ""
    print(f"{op:12s} {100 * n / tot:5.1f}%{extra}")
