"""C5 end to end: qmc_render of the 4K image into pinned host memory (the
render in row bands with each band's D2H overlapping the next band's render,
QMC_RENDER_BANDS = number of bands), host-timed, median of 7; checks the
host image against a device render."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_15584_b200 as q  # noqa: E402

host = torch.empty((2160, 3840), dtype=torch.float32, pin_memory=True).numpy()
for kind in ["pixel-shifted-lattice", "image-plane-halton"]:
    ref = q.render(3840, 2160, 64, kind=kind).cpu().numpy()
    for spp in [16, 64]:
        ref = q.render(3840, 2160, spp, kind=kind).cpu().numpy()
        row = []
        for bands in ["1", "4", "8", "16"]:
            os.environ["QMC_RENDER_BANDS"] = bands
            q.render(3840, 2160, spp, kind=kind, out=host)
            ok = np.array_equal(host.view(np.uint32), ref.view(np.uint32))
            ts = []
            for _ in range(7):
                a = time.perf_counter()
                q.render(3840, 2160, spp, kind=kind, out=host)
                ts.append(time.perf_counter() - a)
            ts.sort()
            row.append("bands=%s %.1f%s" % (bands, 3840 * 2160 * spp / ts[3] / 1e9, "" if ok else " MISMATCH"))
        print(kind[:12], spp, " | ".join(row), flush=True)
os.environ.pop("QMC_RENDER_BANDS", None)
