"""Probe: Halton fills with dims % 32 == 0 (k_tma<HaltonWalk>), Gsamples/s
and fraction of the measured HBM copy peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2307_15584_b200 as q

peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]


def t(fn, samples, k=7):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[len(ev) // 2]
    g = samples / (ms * 1e-3) / 1e9
    return "%.1f Gsamples/s (%.3f ms, %.3f of %.0f GB/s)" % (g, ms, g * 4 / peak, peak)


n = 1 << 24
for d in [32, 64, 256]:
    nn = n if d <= 64 else n // 8
    o = torch.empty((nn, d), dtype=torch.float32, device="cuda")
    for sc in ["linear", "plain", "faure"]:
        print("halton", d, sc, t(lambda: q.halton_fill(nn, d, scramble=sc, out=o), nn * d))
o = torch.empty((1 << 26, 32), dtype=torch.float32, device="cuda")
print("halton 2^26 x 32 linear", t(lambda: q.halton_fill(1 << 26, 32, scramble="linear", out=o), (1 << 26) * 32))
