"""Write-ceiling experiment: store-stream probes vs the C2 fill, same buffer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_15584_b200 as q

n, d = 1 << 28, 32
out = torch.empty((n, d), dtype=torch.float32, device="cuda")
m = q.GeneratorMatrixSet.builtin(d)
B = n * d * 4
def t(fn, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return B / (ms[len(ms)//2] * 1e-3) / 1e9, B / (ms[0] * 1e-3) / 1e9
for rep in range(2):
    for mode in range(6):
        print("probe mode %d: median %.0f GB/s best %.0f" % ((mode,) + t(lambda: q.write_probe(out, mode))))
    print("C2 fill      : median %.0f GB/s best %.0f" % t(lambda: q.sobol_fill(n, d, matrices=m, out=out)))
    print("torch zero_  : median %.0f GB/s best %.0f" % t(lambda: out.zero_()))
