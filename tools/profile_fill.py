"""One warm-up + one measured launch of a hot kernel, for ncu captures.

  ncu --set full --replay-mode application -k regex:<kernel> -s 1 -c 1 \\
      python tools/profile_fill.py --config c2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--launches", type=int, default=2)
a = ap.parse_args()
torch.cuda.set_device(0)
if a.config == "c2":
    n, d = 1 << 28, 32
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    m = q.GeneratorMatrixSet.builtin(d)
    fn = lambda: q.sobol_fill(n, d, matrices=m, out=out)  # noqa: E731
elif a.config in ("c3owen", "c3xor"):
    n, d = 1 << 28, 64
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    m = q.GeneratorMatrixSet.builtin(d)
    seeds = [q.pixel_hash(j, 1, 0x5EED) for j in range(d)]
    sc = "owen" if a.config == "c3owen" else "xor"
    fn = lambda: q.sobol_fill(n, d, matrices=m, scramble=sc, words=seeds, out=out)  # noqa: E731
elif a.config == "c4":
    n, d = 1 << 30, 16
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    g = q.lfsr_generator_vector(0xACE1, d)
    s = [q.pixel_hash(j, 1, 0x5EED) for j in range(d)]
    fn = lambda: q.lattice_fill(n, g, shifts=s, out=out)  # noqa: E731
elif a.config == "c1":
    n = 1 << 24
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    fn = lambda: q.radical_inverse_fill(n, 0, out=out)  # noqa: E731
elif a.config.startswith("halton"):  # halton (2^24 x 32) or halton<dims> (2^29 samples)
    d = int(a.config[6:] or 32)
    n = (1 << 24) if d == 32 else (1 << 29) // d
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    fn = lambda: q.halton_fill(n, d, scramble="linear", out=out)  # noqa: E731
elif a.config in ("sobolowen12", "sobolowen256"):
    d = 12 if a.config.endswith("12") else 256
    n = (1 << 30) // d
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    m = q.GeneratorMatrixSet.builtin(min(d, 64)) if d <= 64 else q.GeneratorMatrixSet.from_columns(
        __import__("numpy").arange(d * 52, dtype="uint32").reshape(d, 52) | 1)
    fn = lambda: q.sobol_fill(n, d, matrices=m, scramble="owen", words=list(range(d)), out=out)  # noqa: E731
elif a.config.startswith("bench-"):
    kern = a.config[len("bench-"):]
    fn = lambda: q.run_bench_kernel(kern, 1 << 28, 32)  # noqa: E731
elif a.config == "integrate":
    fn = lambda: q.integrate("sobol", "product-sine", 1 << 26, 8, "kahan")  # noqa: E731
elif a.config == "c5iph":
    out = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
    fn = lambda: q.render(3840, 2160, 64, kind="image-plane-halton", out=out)  # noqa: E731
elif a.config == "c5hh":
    out = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
    fn = lambda: q.render(3840, 2160, 64, kind="halton-hilbert", out=out)  # noqa: E731
elif a.config.startswith("c5"):
    spp = int(a.config[2:] or 64)
    out = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
    fn = lambda: q.render(3840, 2160, spp, out=out)  # noqa: E731
else:
    raise SystemExit("unknown config")
for _ in range(a.launches):
    fn()
torch.cuda.synchronize()
print("done", a.config)
