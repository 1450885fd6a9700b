import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_15584_b200 as q
g = q.lfsr_generator_vector(0xACE1, 8)
for kind in ["sobol", "halton", "lattice"]:
    for f in ["product-sine", "product-poly"]:
        for n in [1 << 20, 1 << 26, 1 << 28]:
            kw = {"generator": g} if kind == "lattice" else {}
            q.integrate(kind, f, n, 8, **kw)
            t = time.perf_counter(); r = q.integrate(kind, f, n, 8, **kw); dt = time.perf_counter() - t
            print(kind, f, n, "%.1f Gsamples/s  %.2f ms" % (n * 8 / dt / 1e9, dt * 1e3))
