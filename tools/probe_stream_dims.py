import sys; sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2307_15584_b200 as q
for kind in q.SAMPLER_KINDS:
    for dims in (64, 65, 300, 1000, 1001):
        kw = {}
        if kind in ("lattice", "pixel-shifted-lattice"):
            kw["generator"] = q.lfsr_generator_vector(0xACE1, dims)
        if kind in ("halton-hilbert", "pixel-shifted-lattice"):
            kw.update(order=6, pixel=(5, 7))
        if kind == "halton-hilbert":
            kw["spp"] = 5000
        if kind == "image-plane-halton":
            kw.update(width=30, height=20, pixel=(5, 7))
        if kind == "sobol-xor-table":
            kw.update(xor_point_count=64, xor_seed=3)
        try:
            o = q.stream_fill(kind, 3000, dims, **kw); torch.cuda.synchronize()
            r = "ok"
        except Exception as e:
            r = type(e).__name__ + ": " + str(e)[:80]
        print(kind, dims, r)
