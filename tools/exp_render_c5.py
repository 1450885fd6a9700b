"""Probe: BASELINE C5 render rates (3840x2160) per kind / spp / accumulator,
optionally against an alternative libqmcgpu.so (argv[1])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2307_15584_b200 as q

if len(sys.argv) > 1:
    q.LIB_PATH = os.path.abspath(sys.argv[1])
img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")


def t(fn, px, k=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[k // 2]
    return "%.1f" % (px / (ms * 1e-3) / 1e9)


row = []
for kind, spp, acc in [("pixel-shifted-lattice", 1, "kahan"), ("sobol", 1, "kahan"),
                       ("pixel-shifted-lattice", 16, "kahan"), ("pixel-shifted-lattice", 64, "kahan"),
                       ("pixel-shifted-lattice", 256, "kahan"), ("pixel-shifted-lattice", 64, "int"),
                       ("image-plane-halton", 64, "kahan"), ("image-plane-halton", 256, "kahan"),
                       ("halton-hilbert", 64, "kahan"), ("halton", 64, "kahan"), ("sobol", 64, "kahan")]:
    row.append("%s/%d/%s=%s" % (kind[:5], spp, acc, t(lambda: q.render(3840, 2160, spp, kind=kind, accum=acc, out=img), 3840 * 2160 * spp)))
print(os.path.basename(q.LIB_PATH), " ".join(row))
im = q.render(3840, 2160, 64).cpu().numpy()
im2 = q.render(3840, 2160, 64, kind="image-plane-halton").cpu().numpy()
im3 = q.render(3840, 2160, 16, accum="int").cpu().numpy()
print(os.path.basename(q.LIB_PATH), "fnv psl64=%016x iph64=%016x psl16int=%016x" % (q.fnv1a64(im), q.fnv1a64(im2), q.fnv1a64(im3)))
