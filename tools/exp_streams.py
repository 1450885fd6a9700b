"""Stream-fill (make_stream + sample) throughput for every SampleStream kind
at one pixel: 2^24 indices (2^12 for the XOR-table kind) x 4 dims."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402


def t(fn, samples, k=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(k)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[k // 2]
    return "%.1f Gsamples/s (%.3f ms)" % (samples / (ms * 1e-3) / 1e9, ms)


d = 4
g = q.lfsr_generator_vector(0xACE1, d)
xt = q.XorTables.white_noise(d, 1 << 12, 3)
for kind in q.SAMPLER_KINDS:
    n = 1 << 12 if kind == "sobol-xor-table" else 1 << 24
    kw = {}
    if kind in ("lattice", "pixel-shifted-lattice"):
        kw["generator"] = g
    if kind in ("halton-hilbert", "pixel-shifted-lattice", "pixel-random-lattice"):
        kw.update(order=12, pixel=(1000, 700))
    if kind == "halton-hilbert":
        kw["spp"] = n
    if kind == "image-plane-halton":
        kw.update(width=3840, height=2160, pixel=(1000, 700))
    if kind == "sobol-xor-table":
        kw.update(xor_tables=xt, pixel=(17, 5))
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    print(kind, t(lambda: q.stream_fill(kind, n, d, out=out, **kw), n * d))
