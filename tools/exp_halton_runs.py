"""Halton fill throughput vs dims under launch knobs read once per process
(one subprocess per config). argv[1]: comma-separated configs, each
"KEY=VAL+KEY=VAL" (e.g. QMC_HALTON_TILE_WORDS=49152+QMC_HALTON_UNROLL=8)."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2307_15584_b200 as q
def t(fn, samples, k=7):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[len(ev) // 2]
    return samples / (ms * 1e-3) / 1e9
x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
for _ in range(200): x.fill_(1.0)  # clocks up
res = []
for d in %r:
    n = (1 << 29) // d
    o = torch.empty((n, d), dtype=torch.float32, device="cuda")
    res.append("%%d:%%.0f" %% (d, t(lambda: q.halton_fill(n, d, first=1 << 20, scramble="linear", out=o), n * d)))
print(" ".join(res))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dims = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 5, 8, 12, 16, 24, 31, 32, 33, 64]
for cfg in sys.argv[1].split(","):
    env = dict(os.environ)
    for kv in filter(None, cfg.split("+")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CODE % (root, dims)], env=env, capture_output=True, text=True)
    print(cfg, r.stdout.strip(), r.stderr.strip()[-300:])
