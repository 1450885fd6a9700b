"""Summarise an ncu report (raw page) into the metrics DESIGN/profiles cite."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_write.sum.per_second", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")]
    res = {"kernel": name}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            res[k] = (v[i], u[i])
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), n.split("stalled_")[1]))
            except ValueError:
                pass
    tot = sum(x for x, _ in stalls) or 1
    res["top_stalls"] = [(n, round(100 * x / tot, 1)) for x, n in sorted(stalls, reverse=True)[:6]]
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        r = summary(rep)
        print("==", rep)
        for k, val in r.items():
            print("  ", k, val)
