"""Pin the CPU oracle (oracle/qmc_oracle.c) before trusting it.

Each test checks the C restatement against the golden vectors that
tests/golden/make_golden.py recorded from the reference itself, and — when the
reference build is present — against the reference on fresh random probes.
CPU only.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import ptr


def fnv(o, a):
    a = np.ascontiguousarray(a)
    return "%016x" % o.qo_fnv1a64(ptr(a), a.nbytes)


# ------------------------------------------------------------------ unitfloat
def test_map_probes(oracle, golden):
    for u, bits in golden["map_probes"]:
        assert oracle.qo_map_bits(u) == bits, hex(u)


def test_map_range_checksums(oracle, golden):
    for lo, n, h in golden["map_range_fnv"]:
        out = np.empty(n, np.uint32)
        oracle.qo_map_range(lo, n, ptr(out))
        assert fnv(oracle, out) == h


def test_map_random(oracle, golden_arrays):
    u, expect = golden_arrays["map_rand_in"], golden_arrays["map_rand_out"]
    got = np.array([oracle.qo_map_bits(int(x)) for x in u[:8192]], np.uint32)
    np.testing.assert_array_equal(got, expect[:8192])


def test_map_optimal_stratified(oracle):
    """SPEC acceptance 1 on a stratified subset: no binary32 in [0,1) is
    strictly closer to u*2^-32 than map(u); ties go toward zero."""
    rng = np.random.default_rng(7)
    us = np.concatenate([np.arange(0, 1 << 12, dtype=np.uint64),
                         rng.integers(0, 1 << 32, 1 << 14, dtype=np.uint64),
                         np.arange((1 << 32) - 4096, 1 << 32, dtype=np.uint64)])
    for u in us.tolist():
        b = oracle.qo_map_bits(u)
        f = np.uint32(b).view(np.float32)
        assert 0.0 <= f < 1.0
        x = u * 2.0 ** -32
        d = abs(float(f) - x)
        for nb in (b - 1, b + 1):
            if 0 <= nb < 0x3F800000:
                g = float(np.uint32(nb).view(np.float32))
                assert abs(g - x) >= d


def test_brev_clz(oracle, golden):
    for v, r in golden["brev_probes"]:
        assert oracle.qo_brev32(v) == r
    for v, r in golden["clz_probes"]:
        assert oracle.qo_clz32(v) == r


# --------------------------------------------------------------------- primes
def test_primes(oracle, golden_arrays):
    p, mp = C.c_uint32(), C.c_uint32()
    for k in range(1000):
        assert oracle.qo_prime(k, C.byref(p)) == 0 and oracle.qo_prime_max_power(k, C.byref(mp)) == 0
        assert p.value == golden_arrays["primes"][k]
        assert mp.value == golden_arrays["prime_max_powers"][k]
    assert oracle.qo_prime(1000, C.byref(p)) == 3  # out_of_range


# -------------------------------------------------------------------- radical
def test_radical_plain_linear_faure(oracle, golden_arrays, golden):
    n = golden_arrays["radinv_plain"].shape[1]
    for j in range(16):
        b = int(golden_arrays["primes"][j])
        sigma = np.array(golden["faure"][str(b)], np.uint32) if b < 32 else None
        for i in range(0, n, 7):
            assert oracle.qo_radical_inverse_fixed(i, j) == golden_arrays["radinv_plain"][j, i]
            assert (oracle.qo_radical_inverse_linscramble_fixed(i, j, b - 1)
                    == golden_arrays["radinv_linear"][j, i])
            if sigma is not None:
                assert (oracle.qo_radical_inverse_permuted_fixed(i, j, ptr(sigma))
                        == golden_arrays["radinv_faure"][j, i])
    idx = golden_arrays["radinv_big_idx"]
    for j in range(8):
        for k, i in enumerate(idx.tolist()):
            assert oracle.qo_radical_inverse_fixed(i, j) == golden_arrays["radinv_big"][j, k]


def test_base2_is_brev_of_low31(oracle):
    rng = np.random.default_rng(1)
    for i in rng.integers(0, 1 << 32, 4096).tolist() + [0x80000001, 0xFFFFFFFF]:
        assert oracle.qo_radical_inverse_fixed(i, 0) == oracle.qo_brev32(i & 0x7FFFFFFF)


def test_faure(oracle, golden):
    for b in range(2, 32):
        out = np.zeros(b, np.uint32)
        oracle.qo_faure_permutation(b, ptr(out))
        assert out.tolist() == golden["faure"][str(b)]
    assert golden["faure"]["5"] == [0, 3, 2, 1, 4]


def test_tabled(oracle, golden_arrays, golden):
    cases = [("tabled_b3d2", 3, 2, [0, 1, 2]), ("tabled_b5d2", 5, 2, golden["faure"]["5"]),
             ("tabled_b3d4", 3, 4, [0, 1, 2])]
    for name, b, d, sig in cases:
        sigma = np.array(sig, np.uint32)
        table = np.zeros(b ** d, np.uint32)
        assert oracle.qo_tensor_digit_table(ptr(sigma), b, d, ptr(table)) == b ** d
        exp = golden_arrays[name]
        for i in range(exp.size):
            assert oracle.qo_radical_inverse_tabled_fixed(i, b, d, ptr(table), ptr(sigma)) == exp[i]
    t = np.zeros(9, np.uint32)
    oracle.qo_tensor_digit_table(ptr(np.array([0, 1, 2], np.uint32)), 3, 2, ptr(t))
    assert t.tolist() == [0, 3, 6, 1, 4, 7, 2, 5, 8]  # SPEC.md radinv3 table


# ---------------------------------------------------------------------- sobol
def test_sobol_columns(columns64, golden_arrays):
    np.testing.assert_array_equal(columns64, golden_arrays["sobol_columns64"])
    assert hex(columns64[3, 32]) == "0xf80f80d8" and hex(columns64[3, 51]) == "0x25d93000"


def test_sobol_points(oracle, columns64, golden_arrays, golden):
    out = np.zeros((1024, 64), np.uint32)
    oracle.qo_sobol_fill_fixed(0, 1024, 64, ptr(columns64), None, ptr(out))
    np.testing.assert_array_equal(out, golden_arrays["sobol_fixed_1024x64"])
    hi = golden_arrays["sobol_hi_idx"]
    for k, i in enumerate(hi.tolist()):
        oracle.qo_sobol_fill_fixed(i, 1, 64, ptr(columns64), None, ptr(out[0]))
        np.testing.assert_array_equal(out[0], golden_arrays["sobol_hi"][k])
    f = np.zeros((1 << 16, 32), np.uint32)
    oracle.qo_sobol_fill_fixed(0, 1 << 16, 32, ptr(np.ascontiguousarray(columns64[:32])), None, ptr(f))
    m = np.zeros_like(f)
    mv = np.vectorize(oracle.qo_map_bits, otypes=[np.uint32])
    m = mv(f)
    assert fnv(oracle, m) == golden["sobol_f32_65536x32_fnv"]


def test_sobol_xor(oracle, columns64, golden_arrays, golden):
    seeds = golden_arrays["seeds_c3"]
    out = np.zeros((256, 64), np.uint32)
    oracle.qo_sobol_fill_fixed(0, 256, 64, ptr(columns64), ptr(seeds), ptr(out))
    mv = np.vectorize(oracle.qo_map_bits, otypes=[np.uint32])
    np.testing.assert_array_equal(mv(out), golden_arrays["sobol_xor_f32_256x64"].view(np.uint32))


def test_owen_is_nested_uniform(oracle, columns64):
    """Owen scramble (builder-defined) preserves the (0,m)-stratification of
    every 1-D projection and depends on each seed."""
    rng = np.random.default_rng(3)
    seeds = rng.integers(0, 1 << 32, 64, dtype=np.uint64).astype(np.uint32)
    n = 1 << 10
    out = np.zeros((n, 64), np.uint32)
    oracle.qo_sobol_owen_fill_fixed(0, n, 64, ptr(columns64), ptr(seeds), ptr(out))
    for j in range(64):
        for m in (1, 4, 10):
            strata = (out[: 1 << m, j] >> (32 - m))
            assert np.unique(strata).size == 1 << m
    # prefix property: digit k depends only on digits < k and the seed
    for v in rng.integers(0, 1 << 32, 200).tolist():
        s = int(seeds[0])
        for k in (1, 5, 17):
            mask = ~((1 << (32 - k)) - 1) & 0xFFFFFFFF
            w = (v & mask) | (rng.integers(0, 1 << 32) & ~mask & 0xFFFFFFFF)
            assert (oracle.qo_owen_scramble(v, s) & mask) == (oracle.qo_owen_scramble(w, s) & mask)
    assert oracle.qo_owen_scramble(0x12345678, 1) != oracle.qo_owen_scramble(0x12345678, 2)


# -------------------------------------------------------------------- lattice
def test_lattice(oracle, golden_arrays, golden):
    g = np.zeros(16, np.uint32)
    assert oracle.qo_lfsr_generator_vector(0xACE1, 16, ptr(g)) == 0
    np.testing.assert_array_equal(g, golden_arrays["lfsr_ace1_16"])
    assert g[:2].tolist() == [1, 1276675999]
    exp = golden_arrays["lattice_f32_4096x16"].view(np.uint32)
    for i in range(0, 4096, 13):
        for j in range(16):
            assert oracle.qo_map_bits(oracle.qo_lattice_component_fixed(i, int(g[j]))) == exp[i, j]
    for j, x, y, h in golden["pixel_hash_probes"]:
        assert oracle.qo_pixel_hash(j, x, y) == h
    d = np.zeros(16, np.uint32)
    assert oracle.qo_lattice_shift_fixed(5, 7, ptr(g), 16, ptr(d)) == 0
    np.testing.assert_array_equal(d, golden_arrays["lattice_shift_k5_m7"])
    assert oracle.qo_lattice_shift_fixed(1 << 30, 4, ptr(g), 16, ptr(d)) == 4  # overflow


def test_lattice_cp_wrap(oracle, golden_arrays, golden):
    g, s = golden_arrays["lfsr_ace1_16"], golden_arrays["cp_shifts16"]
    first, n = (1 << 32) - 30000, 1 << 16
    i = (np.arange(n, dtype=np.uint64) + first) & 0xFFFFFFFF
    brev = np.vectorize(oracle.qo_brev32, otypes=[np.uint32])(i.astype(np.uint32))
    fx = (brev[:, None].astype(np.uint64) * g[None, :] + s[None, :]) & 0xFFFFFFFF
    out = np.vectorize(oracle.qo_map_bits, otypes=[np.uint32])(fx.astype(np.uint32))
    assert fnv(oracle, out) == golden["lattice_cp_f32_wrap_fnv"]
    for k in range(0, n, 997):
        for j in range(16):
            assert oracle.qo_lattice_cp_fixed(int(i[k]), int(g[j]), int(s[j])) == fx[k, j]


# ------------------------------------------------------- hilbert / enumeration
def test_hilbert(oracle, golden):
    d = C.c_uint64()
    x, y = C.c_uint32(), C.c_uint32()
    for order, grid in golden["hilbert_grids"].items():
        order = int(order)
        for yy, row in enumerate(grid):
            for xx, v in enumerate(row):
                assert oracle.qo_hilbert_index(xx, yy, order, C.byref(d)) == 0 and d.value == v
                assert oracle.qo_hilbert_xy(v, order, C.byref(x), C.byref(y)) == 0
                assert (x.value, y.value) == (xx, yy)
    for px, py, v in golden["phi3_order12"]:
        assert oracle.qo_hilbert_phi3_fixed(px, py, 12) == v
    assert oracle.qo_hilbert_index(0, 0, 0, C.byref(d)) == 2
    assert oracle.qo_hilbert_index(2, 0, 1, C.byref(d)) == 3


def test_halton_enumeration(oracle, golden):
    from oracle import load_oracle  # noqa: F401

    class E(C.Structure):
        _fields_ = [("scale_x", C.c_uint32), ("scale_y", C.c_uint32), ("exp_x", C.c_uint32),
                    ("exp_y", C.c_uint32), ("stride", C.c_uint64), ("crt_x", C.c_uint64),
                    ("crt_y", C.c_uint64)]

    for key, rec in golden["halton_enum"].items():
        w, h = map(int, key.split("x"))
        e = E()
        assert oracle.qo_halton_enum_init(w, h, C.byref(e)) == 0
        assert e.stride == rec["stride"]
        assert [e.exp_x, e.exp_y, e.scale_x, e.scale_y] == rec["exps"]
        for px, py, off in rec["offsets"]:
            assert oracle.qo_halton_enum_offset(C.byref(e), px, py) == off
    r, m = C.c_uint64(), C.c_uint64()
    for p, parts, b, rem, mod in golden["partition"]:
        assert oracle.qo_partition(p, parts, b, C.byref(r), C.byref(m)) == 0
        assert (r.value, m.value) == (rem, mod)
    assert oracle.qo_partition(0, 6, 2, C.byref(r), C.byref(m)) == 1  # ConfigError


# --------------------------------------------------------------------- render
KINDS = {"sobol": 0, "halton": 1, "lattice": 2, "halton-hilbert": 3,
         "pixel-shifted-lattice": 4, "pixel-random-lattice": 5, "image-plane-halton": 6}


@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("accum", ["kahan", "int"])
def test_render64(oracle, golden, columns64, kind, accum):
    img = np.zeros((64, 64), np.float32)
    cols2 = np.ascontiguousarray(columns64[:2])
    assert oracle.qo_render(64, 64, 16, KINDS[kind], 0 if accum == "kahan" else 1, 0,
                            ptr(cols2), ptr(img)) == 0
    assert fnv(oracle, img) == golden["render64_spp16_fnv"]["%s/%s" % (kind, accum)]


def test_scene_value_matches_ref(oracle, ref):
    rng = np.random.default_rng(11)
    for x, y in rng.random((2000, 2)).tolist():
        assert oracle.qo_scene_value(x, y) == ref.ref_scene_value(x, y)


def test_oracle_vs_ref_random_sobol(oracle, ref, columns64):
    rng = np.random.default_rng(5)
    for i in rng.integers(0, 1 << 52, 64, dtype=np.uint64).tolist():
        a = np.zeros(64, np.uint32)
        b = np.zeros(64, np.uint32)
        oracle.qo_sobol_fill_fixed(i, 1, 64, ptr(columns64), None, ptr(a))
        assert ref.ref_sobol_fixed_fill(i, 1, 64, None, ptr(b), 1) == 0
        np.testing.assert_array_equal(a, b)


def test_sobol_fill_f32_port_matches_reference(oracle, ref, columns64):
    """qo_sobol_fill_f32 (bench.py's CPU "port" when the reference build is
    absent) gives the reference's float points bit for bit."""
    from oracle import ptr

    n, dims = 5000, 32
    cols = np.ascontiguousarray(columns64[:dims])
    got = np.zeros((n, dims), np.float32)
    exp = np.zeros((n, dims), np.float32)
    oracle.qo_sobol_fill_f32(12345, n, dims, ptr(cols), None, ptr(got))
    assert ref.ref_sobol_fill(12345, n, dims, None, ptr(exp), 4) == 0
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))
