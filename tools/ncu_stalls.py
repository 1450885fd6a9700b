"""Stall reasons summed over the instructions of one execution count (a loop
body) of an ncu report's SASS page, plus shared-memory wavefronts.

  python tools/ncu_stalls.py rep.ncu-rep <exec_count>[,<exec_count>...]
"""
import csv
import subprocess
import sys
from collections import Counter

rep, keys = sys.argv[1], {int(x) for x in sys.argv[2].split(",")}
rows = list(csv.reader(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
    capture_output=True, text=True).stdout.splitlines()))
h = rows[1]
iE = h.index("Instructions Executed")
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
iw, iwi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
tot, wf, wfi, n = Counter(), 0, 0, 0
for r in rows[2:]:
    try:
        e = int(r[iE] or 0)
    except (ValueError, IndexError):
        continue
    if e not in keys:
        continue
    n += e
    for i in cols:
        tot[h[i]] += int(float(r[i] or 0))
    wf += int(float(r[iw] or 0))
    wfi += int(float(r[iwi] or 0))
s = sum(tot.values())
print("instructions", n, "stall samples", s, "smem wavefronts", wf, "ideal", wfi)
for k, v in tot.most_common(10):
    print("  %-24s %6d  %5.1f%%" % (k, v, 100 * v / max(s, 1)))
