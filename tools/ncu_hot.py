"""Summarise an ncu report's SASS page: total warp instructions, the
instruction mix per execution count (loops), and stall samples.

  python tools/ncu_hot.py gpurun_out/prof_x.ncu-rep [min_share]
"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]
iE, iS = h.index("Instructions Executed"), h.index("Source")
iW = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((r[iS], int(r[iE] or 0), int(r[iW] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(d[1] for d in data)
stall = sum(d[2] for d in data)
print("total warp instructions", tot, "stall samples", stall)
c, w = Counter(), Counter()
for s, n, st in data:
    c[n] += n
    w[n] += st
for n, v in sorted(c.items(), key=lambda x: -x[1])[:12]:
    print("%10d x %3d instr = %5.1f%% of instr, %5.1f%% of stall samples" %
          (n, v // n if n else 0, 100 * v / tot, 100 * w[n] / max(stall, 1)))
if len(sys.argv) > 3:
    keep = {int(x) for x in sys.argv[3].split(",")}
    for s, n, st in data:
        if n in keep:
            print(n, "%-70s" % s[:70], st)
