import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q
def t(fn, B, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[k // 2]
    return "%.0f GB/s" % (B / (ms * 1e-3) / 1e9)
for dims in (3, 5, 12, 48, 100):
    n = (1 << 30) // dims // 4 * 4
    m = q.GeneratorMatrixSet.builtin(min(dims, 64)) if dims <= 64 else q.GeneratorMatrixSet.from_columns(
        __import__("numpy").arange(dims * 52, dtype="uint32").reshape(dims, 52) | 1)
    out = torch.empty((n, dims), dtype=torch.float32, device="cuda")
    B = out.numel() * 4
    print(dims, "plain", t(lambda: q.sobol_fill(n, dims, matrices=m, out=out), B),
          "owen", t(lambda: q.sobol_fill(n, dims, matrices=m, scramble="owen", words=list(range(dims)), out=out), B))
    del out

for dims in (3, 5, 12, 48, 100):
    n = (1 << 30) // dims // 4 * 4
    g = q.lfsr_generator_vector(0xACE1, dims)
    out = torch.empty((n, dims), dtype=torch.float32, device="cuda")
    B = out.numel() * 4
    print(dims, "lattice", t(lambda: q.lattice_fill(n, g, out=out), B),
          "cp", t(lambda: q.lattice_fill(n, g, shifts=list(range(dims)), out=out), B))
    del out
