"""Lattice fill (plain and CP-shifted) write rate vs dims."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402


def t(fn, B, k=5):
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
    return "%.0f" % (B / (ms * 1e-3) / 1e9)


x = torch.empty(1 << 30, device="cuda")
for _ in range(200):
    x.fill_(1)
del x
for dims in (3, 5, 6, 7, 10, 12, 20, 24, 31, 40, 48, 96, 100, 200):
    n = (1 << 30) // dims // 4 * 4
    g = q.lfsr_generator_vector(0xACE1, dims)
    out = torch.empty((n, dims), dtype=torch.float32, device="cuda")
    B = out.numel() * 4
    print(dims, "lattice GB/s", t(lambda: q.lattice_fill(n, g, out=out), B),
          "cp", t(lambda: q.lattice_fill(n, g, shifts=list(range(dims)), out=out), B), flush=True)
    del out
