"""A/B of the level-table Halton fill (k_halton_lv) against the k_tma walk
(QMC_HALTON_NO_LV=1) at dims % 32 == 0: bit-identity of the two and
Gsamples/s (CUDA events, median of 7)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q

# argv: [alternative libqmcgpu.so] [--quick: timings only, linear scramble]
quick = "--quick" in sys.argv
alt = [a for a in sys.argv[1:] if a != "--quick"]
if alt:
    q.LIB_PATH = os.path.abspath(alt[0])


def t(fn, samples, k=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[len(ev) // 2]
    return samples / (ms * 1e-3) / 1e9, ms


def both(fn):
    os.environ.pop("QMC_HALTON_NO_LV", None)
    a = fn()
    os.environ["QMC_HALTON_NO_LV"] = "1"
    b = fn()
    os.environ.pop("QMC_HALTON_NO_LV", None)
    return a, b


for first in ([] if quick else [0, 1 << 20, 3486784401 - 77777, 2**31 - 5000, 2**32 - 100000]):
    for sc in ["plain", "linear", "faure"]:
        a, b = both(lambda: q.halton_fill(300000, 32, first=first, scramble=sc, fixed=True).cpu())
        print("identity first=%d %s: %s" % (first, sc, bool(torch.equal(a, b))), flush=True)
n, d = 1 << 24, 32
out = torch.empty((n, d), dtype=torch.float32, device="cuda")
for sc in (["linear"] if quick else ["linear", "plain", "faure"]):
    for lv in ([True] if quick else [True, False]):
        if lv:
            os.environ.pop("QMC_HALTON_NO_LV", None)
        else:
            os.environ["QMC_HALTON_NO_LV"] = "1"
        g, ms = t(lambda: q.halton_fill(n, d, first=1 << 20, scramble=sc, out=out), n * d)
        print("halton 2^24x32 %s %s: %.1f Gsamples/s %.3f ms (%.3f of 6554.2 GB/s)"
              % (sc, "lv" if lv else "k_tma", g, ms, g * 4 / 6554.2), flush=True)
os.environ.pop("QMC_HALTON_NO_LV", None)
