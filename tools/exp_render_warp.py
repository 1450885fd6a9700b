import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2307_15584_b200 as q
for kind in ["pixel-shifted-lattice", "sobol", "image-plane-halton", "halton-hilbert"]:
    fn = lambda: q.render(64, 64, 65536, kind=kind)
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(kind, "%.1f G pixel-samples/s" % (64*64*65536/ms/1e6))
