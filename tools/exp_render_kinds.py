"""4K render throughput for every sampler kind at 64 spp (Kahan)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
for kind in q.SAMPLER_KINDS:
    fn = lambda: q.render(3840, 2160, 64, kind=kind, out=img)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(5)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[2]
    print("%-22s %.1f G pixel-samples/s" % (kind, 3840 * 2160 * 64 / ms / 1e6))
