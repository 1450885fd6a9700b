"""Integration throughput (host-timed calls, median of 7 after 2 warm-ups)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

if len(sys.argv) > 1:  # an alternative libqmcgpu.so (A/B)
    q.LIB_PATH = os.path.abspath(sys.argv[1])
n, d = 1 << 26, 8
for kind in ["sobol", "halton", "lattice", "pixel-shifted-lattice"]:
    kw = {"generator": q.lfsr_generator_vector(0xACE1, d)} if "lattice" in kind else {}
    if kind == "pixel-shifted-lattice":
        kw.update(pixel=(5, 9), order=12)
    for f in ["product-sine", "product-poly"]:
        fn = lambda: q.integrate(kind, f, n, d, "kahan", **kw)  # noqa: E731
        est = fn()
        fn()
        ts = []
        for _ in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print("%-22s %-13s %.1f Gsamples/s  estimate %r" % (kind, f, n * d / ts[3] / 1e9,
                                                            getattr(est, "estimate", est)))
