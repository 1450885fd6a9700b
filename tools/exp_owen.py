import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q
def t(fn, B, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return "median %.0f GB/s best %.0f" % (B / (ms[len(ms)//2] * 1e-3) / 1e9, B / (ms[0] * 1e-3) / 1e9)
tag = os.environ.get("QMCGPU_LIB", "lk")
m64 = q.GeneratorMatrixSet.builtin(64)
seeds = [q.pixel_hash(j, 1, 0x5EED) for j in range(64)]
out = torch.empty((1 << 27, 64), dtype=torch.float32, device="cuda")
B = out.numel() * 4
for r in range(3):
    print(tag[-14:], "owen", t(lambda: q.sobol_fill(1 << 27, 64, matrices=m64, scramble="owen", words=seeds, out=out), B))
