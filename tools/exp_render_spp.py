import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2307_15584_b200 as q
img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
for spp in (1, 2, 4, 8, 16, 64, 256):
    fn = lambda: q.render(3840, 2160, spp, out=img)
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[2]
    print("spp", spp, "%.1f G pixel-samples/s (%.3f ms)" % (3840*2160*spp/ms/1e6, ms))
