"""Small calls of every kernel family, for compute-sanitizer (memcheck /
racecheck / initcheck) runs: ragged sizes, tails, both lane widths."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2307_15584_b200 as q

torch.cuda.set_device(0)
for dims in (1, 3, 4, 8, 16, 32, 48, 64):
    for first, n in ((0, 777), (12345, 1000), ((1 << 52) - 500, 500)):
        q.sobol_fill(n, dims, first=first)
        q.sobol_fill(n, dims, first=first, scramble="xor", words=list(range(dims)))
        q.sobol_fill(n, dims, first=first, scramble="owen", words=list(range(dims)), fixed=True)
    g = [2 * k + 1 for k in range(dims)]
    q.lattice_fill(999, g, first=(1 << 32) - 100, shifts=list(range(dims)))
    q.halton_fill(333, dims, first=77, scramble="faure")
for n, dims in ((148 * 512 * 2 + 77, 32), (3000, 64), (5000, 96), (70000, 31), (9000, 2)):
    q.halton_fill(n, dims, first=3486784401 - 2000, scramble="linear")  # runs / TMA column blocks
    q.halton_fill(n, dims, first=5, fixed=True)
if os.environ.get("QMC_SANITIZE_HALTON_ONLY"):
    torch.cuda.synchronize()
    print("sanitize smoke done")
    sys.exit(0)
q.radical_inverse_fill(1001, 0)
q.radical_inverse_fill(1001, 5, scramble="linear", factor=3)
q.map_u32_to_unifloat(torch.arange(1000, dtype=torch.int32, device="cuda"))
for kind in q.SAMPLER_KINDS:
    kw = {}
    if kind in ("lattice", "pixel-shifted-lattice"):
        kw["generator"] = q.lfsr_generator_vector(0xACE1, 3)
    if kind in ("halton-hilbert", "pixel-shifted-lattice"):
        kw.update(order=6, pixel=(5, 7))
    if kind == "halton-hilbert":
        kw["spp"] = 50
    if kind == "image-plane-halton":
        kw.update(width=30, height=20, pixel=(5, 7))
    if kind == "sobol-xor-table":
        kw.update(xor_point_count=64, xor_seed=3)
    q.stream_fill(kind, 50, 3, **kw)
    q.render(37, 23, 5, kind=kind, seed=2)
    q.render(37, 23, 5, kind=kind, accum="int", rows=(3, 11))
    if kind != "sobol-xor-table":
        q.integrate(kind, "product-sine", 5000, 3, stream_dims=3, **kw) if kind != "halton-hilbert" else None
    acc = q.render_partial(37, 23, 5, 1, 2, kind=kind)
    q.render_finalize(acc, 5)
# spp >= 32: the phi_3 tables bulk-copied per CTA (image-plane Halton,
# halton, halton-hilbert incremental path); a host image above 2^20 pixels
# (banded render with overlapped D2H)
for kind in ("image-plane-halton", "halton", "halton-hilbert", "pixel-shifted-lattice"):
    q.render(96, 80, 64, kind=kind)
host = np.empty((1100, 1000), np.float32)
q.render(1000, 1100, 8, out=host)
pts = q.sobol_fill(300, 5).contiguous()
q.l2_star_discrepancy(pts)
q.min_toroidal_distance(pts)
q.check_1d_stratification("sobol", 1, 10, 4)
t = q.XorTables.white_noise(3, 128, 1)
q.stream_fill("sobol-xor-table", 100, 3, xor_tables=t, pixel=(3, 4))
out = np.empty((5000, 16), np.float32)
q.sobol_fill(5000, 16, out=out)
torch.cuda.synchronize()
print("sanitize smoke done")
