"""Throughput survey of every public fill/stream/render/integrate entry (one B200)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q

def t(fn, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[k // 2]

rows = []
buf = torch.empty(1 << 31, dtype=torch.float32, device="cuda")  # 8 GiB scratch
def fill(name, n, dims, fn):
    ms = t(lambda: fn(buf[: n * dims]))
    rows.append((name, n, dims, n * dims / ms / 1e6, n * dims * 4 / ms / 1e6))

m = {d: q.GeneratorMatrixSet.builtin(d) for d in (1, 3, 5, 16, 32, 48, 64)}
for d in (1, 3, 5, 16, 32, 48, 64):
    n = (1 << 30) // d
    fill("sobol", n, d, lambda o: q.sobol_fill(n, d, matrices=m[d], out=o))
    fill("sobol owen", n, d, lambda o: q.sobol_fill(n, d, matrices=m[d], scramble="owen", words=list(range(d)), out=o))
    g = [2 * k + 1 for k in range(d)]
    fill("lattice cp", n, d, lambda o: q.lattice_fill(n, g, shifts=list(range(d)), out=o))
for d in (1, 8, 32):
    n = (1 << 27) // d
    fill("halton plain", n, d, lambda o: q.halton_fill(n, d, out=o))
    fill("halton linear", n, d, lambda o: q.halton_fill(n, d, scramble="linear", out=o))
for kind in ("pixel-shifted-lattice", "pixel-random-lattice", "image-plane-halton", "halton-hilbert"):
    kw = {"pixel": (100, 200)}
    if kind == "pixel-shifted-lattice": kw.update(order=12, generator=q.lfsr_generator_vector(0xACE1, 8))
    if kind == "halton-hilbert": kw.update(order=12, spp=1 << 24)
    if kind == "image-plane-halton": kw.update(width=3840, height=2160)
    n = 1 << 24
    fill("stream " + kind, n, 8, lambda o: q.stream_fill(kind, n, 8, out=o, **kw))
print("%-34s %12s %5s %14s %10s" % ("entry", "points", "dims", "Gsamples/s", "GB/s"))
for r in rows:
    print("%-34s %12d %5d %14.1f %10.0f" % r)
del buf
torch.cuda.empty_cache()
img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
for kind in q.SAMPLER_KINDS:
    for accum in ("kahan", "int"):
        ms = t(lambda: q.render(3840, 2160, 64, kind=kind, accum=accum, seed=1, out=img), 3)
        print("render 4K@64 %-24s %-6s %8.1f G px-samples/s" % (kind, accum, 3840 * 2160 * 64 / ms / 1e6))
g8 = q.lfsr_generator_vector(0xACE1, 8)
for kind in ("sobol", "lattice", "halton", "pixel-random-lattice"):
    for f in ("product-sine", "product-poly", "indicator"):
        import time
        kw = {"generator": g8} if kind == "lattice" else {}
        q.integrate(kind, f, 1 << 26, 8, **kw)
        a = time.perf_counter(); q.integrate(kind, f, 1 << 26, 8, **kw); dt = time.perf_counter() - a
        print("integrate 2^26x8 %-22s %-13s %8.1f Gsamples/s" % (kind, f, (1 << 26) * 8 / dt / 1e9))
