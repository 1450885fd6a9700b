import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2307_15584_b200 as q
def t(fn, B, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[k // 2]
    return "%.0f" % (B / (ms * 1e-3) / 1e9)
x = torch.empty(1 << 30, device="cuda")
for _ in range(200): x.fill_(1)
del x
DIMS = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 20, 24, 31, 32, 40, 48, 64, 96, 100, 128, 200, 256]
for dims in DIMS:
    n = (1 << 30) // dims // 4 * 4
    m = q.GeneratorMatrixSet.builtin(min(dims, 64)) if dims <= 64 else q.GeneratorMatrixSet.from_columns(
        np.arange(dims * 52, dtype="uint32").reshape(dims, 52) | 1)
    out = torch.empty((n, dims), dtype=torch.float32, device="cuda")
    B = out.numel() * 4
    print(dims, "sobol GB/s", t(lambda: q.sobol_fill(n, dims, matrices=m, out=out), B),
          "owen", t(lambda: q.sobol_fill(n, dims, matrices=m, scramble="owen", words=list(range(dims)), out=out), B), flush=True)
    del out
