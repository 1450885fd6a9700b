"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libqmcref.so, compiled from
/root/reference/proj/src by oracle/Makefile) and records known-answer vectors
and checksums. Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

Outputs (committed): golden.json (scalars, checksums, small lists) and
golden.npz (uint32/float arrays). Tests read only these files at run time.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import ctypes as C  # noqa: E402

from oracle import load_ref, ptr  # noqa: E402

ref = load_ref()
REF_DATA = "/root/reference/proj/data/joe-kuo-64.txt"


def ok(rc):
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())


def fnv(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % ref.ref_fnv1a64(ptr(a), a.nbytes)


def main() -> None:
    G: dict = {}
    A: dict = {}

    # ---- direction numbers (public Joe-Kuo data, first 64 dims) as rows
    rows = []
    with open(REF_DATA) as f:
        next(f)
        for line in f:
            t = line.split()
            if not t:
                continue
            d, s, a = int(t[0]), int(t[1]), int(t[2])
            rows.append([d, s, a, [int(x) for x in t[3:3 + s]]])
    G["direction_numbers"] = rows

    # ---- unitfloat
    probes = [0, 1, 2, 3, 0x80000000, 0xFFFFFFFF, 0xFFFFFF7F, 0xFFFFFF80, 0x01000100,
              0x01000101, 0x01000180, 0x00FFFFFF, 0x01000000, 0x03FFFFFF, 0x7FFFFFFF,
              0x3F800000, 0xDEADBEEF]
    G["map_probes"] = [[u, ref.ref_map_bits(u)] for u in probes]
    for lo, n in [(0, 1 << 24), (0xFF000000, 1 << 24)]:
        out = np.empty(n, np.uint32)
        ref.ref_map_range(lo, n, ptr(out))
        G.setdefault("map_range_fnv", []).append([lo, n, fnv(out)])
    rng = np.random.default_rng(2307_15584)
    u = rng.integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32)
    mu = np.empty_like(u)
    ref.ref_map_bulk(ptr(u), ptr(mu), u.size)
    A["map_rand_in"], A["map_rand_out"] = u, mu
    G["brev_probes"] = [[v, ref.ref_bit_reverse32(v)] for v in [0, 1, 0xF00F, 0x12345678]]
    G["clz_probes"] = [[v, ref.ref_clz32(v)] for v in [0, 1, 0x80000000, 0x00010000]]

    # ---- primes
    pr = np.zeros(1000, np.uint32)
    mp = np.zeros(1000, np.uint32)
    for k in range(1000):
        a, b = C.c_uint32(), C.c_uint32()
        ok(ref.ref_prime(k, C.byref(a)))
        ok(ref.ref_prime_max_power(k, C.byref(b)))
        pr[k], mp[k] = a.value, b.value
    A["primes"], A["prime_max_powers"] = pr, mp

    # ---- radical inverse: plain / linear(b-1) / faure, dims 0..15
    n = 4096
    for mode, name in [(0, "radinv_plain"), (1, "radinv_linear"), (2, "radinv_faure")]:
        out = np.zeros((16, n), np.uint32)
        for j in range(16):
            ok(ref.ref_radical_fixed_fill(0, n, j, mode, int(pr[j]) - 1, ptr(out[j])))
        A[name] = out
    big = rng.integers(0, 1 << 32, size=2048, dtype=np.uint64).astype(np.uint32)
    out = np.zeros((8, big.size), np.uint32)
    for j in range(8):
        for k, i in enumerate(big):
            ok(ref.ref_radical_fixed_fill(int(i), 1, j, 0, 0, ptr(out[j, k:k + 1])))
    A["radinv_big_idx"], A["radinv_big"] = big, out
    faure = {}
    for b in range(2, 32):
        p = np.zeros(b, np.uint32)
        ok(ref.ref_faure_permutation(b, ptr(p)))
        faure[str(b)] = p.tolist()
    G["faure"] = faure
    for which, name in [(0, "tabled_b3d2"), (1, "tabled_b5d2"), (2, "tabled_b3d4")]:
        o = np.zeros(n, np.uint32)
        ok(ref.ref_radical_tabled_fixed_fill(0, n, which, ptr(o)))
        A[name] = o
    th = np.zeros((512, 32), np.uint32)
    ok(ref.ref_tabled_halton_fixed_fill(1000, 512, 32, ptr(th)))
    A["tabled_halton32_from1000"] = th

    # ---- sobol
    cols = np.zeros((64, 52), np.uint32)
    ok(ref.ref_build_matrices_builtin(64, ptr(cols)))
    A["sobol_columns64"] = cols
    pts = np.zeros((1024, 64), np.uint32)
    ok(ref.ref_sobol_fixed_fill(0, 1024, 64, None, ptr(pts), 1))
    A["sobol_fixed_1024x64"] = pts
    hi = (rng.integers(0, 1 << 52, size=512, dtype=np.uint64))
    hi[:4] = [(1 << 52) - 1, (1 << 32), (1 << 32) - 1, (1 << 40) + 12345]
    hv = np.zeros((512, 64), np.uint32)
    for k, i in enumerate(hi):
        ok(ref.ref_sobol_fixed_fill(int(i), 1, 64, None, ptr(hv[k]), 1))
    A["sobol_hi_idx"], A["sobol_hi"] = hi, hv
    f32 = np.zeros((1 << 16, 32), np.float32)
    ok(ref.ref_sobol_fill(0, 1 << 16, 32, None, ptr(f32), 8))
    G["sobol_f32_65536x32_fnv"] = fnv(f32)
    scr = np.array([ref.ref_pixel_hash(j, 1, 0x5EED) for j in range(64)], np.uint32)
    A["seeds_c3"] = scr
    xf = np.zeros((4096, 64), np.float32)
    ok(ref.ref_sobol_fill(0, 4096, 64, ptr(scr), ptr(xf), 8))
    G["sobol_xor_f32_4096x64_fnv"] = fnv(xf)
    A["sobol_xor_f32_256x64"] = xf[:256].copy()

    # ---- lattice
    g16 = np.zeros(16, np.uint32)
    ok(ref.ref_lfsr_generator_vector(0xACE1, 16, ptr(g16)))
    A["lfsr_ace1_16"] = g16
    G["pixel_hash_probes"] = [[j, x, y, ref.ref_pixel_hash(j, x, y)]
                              for (j, x, y) in [(0, 0, 0), (1, 2, 3), (7, 3839, 2159),
                                                (63, 1, 0x5EED)]]
    lat = np.zeros((4096, 16), np.float32)
    ok(ref.ref_lattice_fill(0, 4096, 16, ptr(g16), None, ptr(lat), 1))
    A["lattice_f32_4096x16"] = lat
    cp = np.array([ref.ref_pixel_hash(j, 1, 0x5EED) for j in range(16)], np.uint32)
    A["cp_shifts16"] = cp
    latc = np.zeros((1 << 16, 16), np.float32)
    ok(ref.ref_lattice_fill((1 << 32) - 30000, 1 << 16, 16, ptr(g16), ptr(cp), ptr(latc), 8))
    G["lattice_cp_f32_wrap_fnv"] = fnv(latc)
    dl = np.zeros(16, np.uint32)
    ok(ref.ref_lattice_shift_fixed(5, 7, ptr(g16), 16, ptr(dl)))
    A["lattice_shift_k5_m7"] = dl

    # ---- hilbert / pixel enumeration
    hil = {}
    for order in (1, 2, 3, 4):
        m = np.zeros((1 << order, 1 << order), np.uint64)
        for x in range(1 << order):
            for y in range(1 << order):
                d = C.c_uint64()
                ok(ref.ref_hilbert_index(x, y, order, C.byref(d)))
                m[y, x] = d.value
        hil[str(order)] = m.tolist()
    G["hilbert_grids"] = hil
    phi = []
    for (x, y) in [(0, 0), (1, 0), (0, 1), (3839, 2159), (1000, 2000), (4095, 4095)]:
        o = C.c_uint32()
        ok(ref.ref_hilbert_phi3_fixed(x, y, 12, C.byref(o)))
        phi.append([x, y, o.value])
    G["phi3_order12"] = phi
    he = {}
    for (w, h) in [(2, 3), (4, 9), (5, 7), (16, 27), (3840, 2160), (64, 64)]:
        offs = []
        for (px, py) in [(0, 0), (1, 0), (w - 1, h - 1), (w // 2, h // 3)]:
            off, st = C.c_uint64(), C.c_uint64()
            ex = np.zeros(4, np.uint32)
            ok(ref.ref_halton_pixel_enum(w, h, px, py, C.byref(off), C.byref(st), ptr(ex)))
            offs.append([px, py, off.value])
        he["%dx%d" % (w, h)] = {"stride": st.value, "exps": ex.tolist(), "offsets": offs}
    G["halton_enum"] = he
    parts = []
    for (p, P_, b) in [(0, 2, 2), (1, 2, 2), (1, 4, 2), (3, 8, 2), (2, 9, 3), (5, 27, 3)]:
        r, m = C.c_uint64(), C.c_uint64()
        ok(ref.ref_partition(p, P_, b, C.byref(r), C.byref(m)))
        parts.append([p, P_, b, r.value, m.value])
    G["partition"] = parts

    # ---- stream façade (every kind except xor-table, float bits)
    streams = {}
    for kind, extra in [("sobol", {}), ("halton", {}), ("lattice", {}),
                        ("halton-hilbert", {"px": 3, "py": 5, "order": 4, "spp": 16}),
                        ("pixel-shifted-lattice", {"px": 3, "py": 5, "order": 12}),
                        ("pixel-random-lattice", {"px": 3, "py": 5}),
                        ("image-plane-halton", {"px": 3, "py": 5, "w": 64, "h": 64})]:
        dims = 2 if kind != "image-plane-halton" else 6
        nn = 256 if kind != "halton-hilbert" else 16
        o = np.zeros((nn, dims), np.uint32)
        ok(ref.ref_stream_fill(kind.encode(), dims, 0, b"plain", extra.get("px", 0),
                               extra.get("py", 0), extra.get("order", 1), extra.get("spp", 1),
                               extra.get("w", 0), extra.get("h", 0), 0, nn, ptr(o)))
        A["stream_" + kind.replace("-", "_")] = o
        streams[kind] = extra
    G["streams"] = streams

    # ---- render goldens (glibc sin: the GPU box runs the same image)
    rend = {}
    for kind in ["pixel-shifted-lattice", "image-plane-halton", "sobol", "pixel-random-lattice",
                 "lattice", "halton", "halton-hilbert"]:
        for accum in ["kahan", "int"]:
            img = np.zeros((64, 64), np.float32)
            ok(ref.ref_render(64, 64, 16, kind.encode(), accum.encode(), 0, 8, ptr(img)))
            rend["%s/%s" % (kind, accum)] = fnv(img)
            A["render64_%s_%s" % (kind.replace("-", "_"), accum)] = img
    G["render64_spp16_fnv"] = rend
    img = np.zeros((2160, 3840), np.float32)
    r4k = {}
    for spp, accum in [(1, "kahan"), (16, "kahan"), (64, "int")]:
        ok(ref.ref_render(3840, 2160, spp, b"pixel-shifted-lattice", accum.encode(), 0, 8,
                          ptr(img)))
        r4k["%d/%s" % (spp, accum)] = fnv(img)
    G["render4k_psl_fnv"] = r4k

    # ---- reference bench checksums (bench.cpp:79-150) at a small count
    bc = {}
    for k in ["sobol", "halton", "halton-tabled", "lattice", "pixel-shifted-lattice",
              "pixel-random-lattice"]:
        cps, cs = C.c_double(), C.c_uint64()
        ok(ref.ref_run_bench_kernel(k.encode(), 1 << 16, 32, C.byref(cps), C.byref(cs)))
        bc[k] = "%016x" % cs.value
    G["bench_checksums_65536x32"] = bc

    # ---- integrate (quality.cpp:214-282); the shim builds the stream like
    # the CLI: lattice g = lfsr(0xace1, max(dims,2)), sobol scrambles =
    # pixel_hash(j, seed, 0x5eed) when seed != 0 (qmckit.cpp:110-119)
    integ = []
    for kind, seed in [("sobol", 0), ("sobol", 7), ("lattice", 0), ("halton", 0),
                       ("pixel-random-lattice", 0)]:
        for f in ["product-sine", "product-poly", "indicator"]:
            for accum in ["kahan", "int"]:
                for dims, n in [(3, 10000), (5, (1 << 20) + 5)]:
                    e = C.c_double()
                    ok(ref.ref_integrate(kind.encode(), dims, seed, f.encode(), n, accum.encode(),
                                         8, C.byref(e)))
                    integ.append([kind, seed, f, accum, dims, n, e.value])
    G["integrate"] = integ

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **A)
    print("wrote golden.json / golden.npz")


if __name__ == "__main__":
    main()
