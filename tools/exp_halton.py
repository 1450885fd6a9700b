import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q
def t(fn, samples, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[len(ev) // 2]
    return "%.1f Gsamples/s (%.2f ms)" % (samples / (ms * 1e-3) / 1e9, ms)
n, d = 1 << 24, 32
out = torch.empty((n, d), dtype=torch.float32, device="cuda")
for sc in ["plain", "linear", "faure"]:
    print("halton", sc, t(lambda: q.halton_fill(n, d, first=1 << 20, scramble=sc, out=out), n * d))
for d2 in [1, 4, 8, 16, 64, 256]:
    o2 = torch.empty((n if d2 <= 64 else n // 8, d2), dtype=torch.float32, device="cuda")
    print("halton dims", d2, t(lambda: q.halton_fill(o2.shape[0], d2, out=o2), o2.numel()))
o1 = torch.empty(n * 4, dtype=torch.float32, device="cuda")
for pi in [1, 30, 700]:
    print("radical prime", pi, t(lambda: q.radical_inverse_fill(n * 4, pi, out=o1), n * 4))
img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
for kind in ["image-plane-halton", "halton", "halton-hilbert", "pixel-shifted-lattice"]:
    print("render", kind, t(lambda: q.render(3840, 2160, 64, kind=kind, out=img), 3840 * 2160 * 64))
