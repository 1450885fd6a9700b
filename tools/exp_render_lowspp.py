"""4K render throughput at low spp for a few sampler kinds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
x = torch.empty(1 << 30, device="cuda")
for _ in range(200):
    x.fill_(1)
del x
for kind in ["pixel-shifted-lattice", "image-plane-halton", "sobol", "halton"]:
    for spp in (1, 2, 4):
        fn = lambda: q.render(3840, 2160, spp, kind=kind, out=img)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(9)]
        for a, b in ev:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)[4]
        print("%-22s spp %d  %.1f G pixel-samples/s (%.3f ms)" % (kind, spp, 3840 * 2160 * spp / ms / 1e6, ms))
