"""C1 (vdc 2^24 x 1) as bench.py times it: a CUDA graph of 12 fills over 4
rotating 64 MiB buffers; prints the per-launch time and TB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

n1 = 1 << 24
o1 = [torch.empty(n1, dtype=torch.float32, device="cuda") for _ in range(4)]
q.radical_inverse_fill(n1, 0, out=o1[0])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.graph(g, stream=cap):
    for k in range(12):
        q.radical_inverse_fill(n1, 0, out=o1[k % 4], stream=cap.cuda_stream)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 12)
ts.sort()
us = ts[len(ts) // 2] * 1e3
print("vdc per launch %.2f us, %.0f GB/s" % (us, n1 * 4 / (us * 1e-6) / 1e9))
