"""Halton fills with dims % 32 == 0 beyond 32 (the level-table fill takes the
leading column blocks whose tables fit, the k_tma walk the rest) against the
k_tma walk alone (QMC_HALTON_NO_LV=1): bit-identity and Gsamples/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q

if len(sys.argv) > 1:  # an alternative libqmcgpu.so (A/B)
    q.LIB_PATH = os.path.abspath(sys.argv[1])


def t(fn, samples, k=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[len(ev) // 2]
    return samples / (ms * 1e-3) / 1e9


for d in [64, 96, 128, 256]:
    n = (1 << 29) // d
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    row = []
    res = {}
    for lv in [True, False]:
        if lv:
            os.environ.pop("QMC_HALTON_NO_LV", None)
        else:
            os.environ["QMC_HALTON_NO_LV"] = "1"
        res[lv] = q.halton_fill(200000, d, first=3486784401 - 70000, scramble="linear", fixed=True).cpu()
        row.append("%s %.1f" % ("lv+tma" if lv else "tma", t(lambda: q.halton_fill(n, d, scramble="linear", out=out), n * d)))
    os.environ.pop("QMC_HALTON_NO_LV", None)
    print("dims %d: %s identical=%s" % (d, " | ".join(row), bool(torch.equal(res[True], res[False]))), flush=True)
