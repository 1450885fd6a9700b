"""Compare fast-fill lane widths (run twice: QMCGPU_FAST_DPL=4 / default 8)."""
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
tag = os.environ.get("QMCGPU_FAST_DPL", "8")
out = torch.empty(1 << 33, dtype=torch.float32, device="cuda")   # 32 GiB
B = out.numel() * 4
m32 = q.GeneratorMatrixSet.builtin(32); m64 = q.GeneratorMatrixSet.builtin(64)
seeds = [q.pixel_hash(j, 1, 0x5EED) for j in range(64)]
g = q.lfsr_generator_vector(0xACE1, 16); s = [q.pixel_hash(j, 1, 0x5EED) for j in range(16)]
print(tag, "C2 sobol32   ", t(lambda: q.sobol_fill(1 << 28, 32, matrices=m32, out=out), B))
print(tag, "sobol64 xor  ", t(lambda: q.sobol_fill(1 << 27, 64, matrices=m64, scramble="xor", words=seeds, out=out), B))
print(tag, "sobol64 owen ", t(lambda: q.sobol_fill(1 << 27, 64, matrices=m64, scramble="owen", words=seeds, out=out), B))
print(tag, "lattice16 cp ", t(lambda: q.lattice_fill(1 << 29, g, shifts=s, out=out), B))
print(tag, "probe v8     ", t(lambda: q.write_probe(out, 2), B))
