"""GPU parity: the CUDA path (through the C-ABI) against the oracle, the
reference build and the golden fixtures. Bit-exact for every integer / float
point set; <= 1e-6 relative for the render (north_star tolerance)."""
import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_15584_b200 as q  # noqa: E402
from oracle import ptr  # noqa: E402


def u32(t):
    return t.cpu().numpy().view(np.uint32) if hasattr(t, "cpu") else np.asarray(t).view(np.uint32)


def fnv(o, a):
    a = np.ascontiguousarray(a)
    return "%016x" % o.qo_fnv1a64(ptr(a), a.nbytes)


@pytest.fixture(scope="module")
def mapv(oracle):
    return np.vectorize(oracle.qo_map_bits, otypes=[np.uint32])


# ------------------------------------------------------------------ map
def test_map_exhaustive_selfcheck():
    """SPEC acceptance 1 on the device: all 2^32 inputs equal the reference formula."""
    assert q.map_selfcheck() == 0


def test_map_vs_golden(golden_arrays, golden):
    u = torch.from_numpy(golden_arrays["map_rand_in"].view(np.int32)).cuda()
    got = u32(q.map_u32_to_unifloat(u))
    np.testing.assert_array_equal(got, golden_arrays["map_rand_out"])
    probes = np.array([p[0] for p in golden["map_probes"]], np.uint32)
    got = q.map_u32_to_unifloat(probes).view(np.uint32)
    assert got.tolist() == [p[1] for p in golden["map_probes"]]


def test_map_range_checksums(golden, oracle):
    for lo, n, h in golden["map_range_fnv"]:
        x = (torch.arange(n, dtype=torch.int64, device="cuda") + lo).to(torch.int64)
        x = (x & 0xFFFFFFFF).to(torch.int64)
        xi = torch.where(x >= 2**31, x - 2**32, x).to(torch.int32)
        assert fnv(oracle, u32(q.map_u32_to_unifloat(xi))) == h


# ------------------------------------------------------------- C1: vdc
def test_vdc_c1_full(oracle, mapv):
    n = 1 << 24
    fx = u32(q.radical_inverse_fill(n, 0, fixed=True))
    i = np.arange(n, dtype=np.uint64)
    exp = np.zeros(n, np.uint32)
    # bit-reverse of i & 0x7fffffff (verified identity, tests/test_oracle.py)
    v = (i & 0x7FFFFFFF).astype(np.uint32)
    for k in range(32):
        exp |= ((v >> np.uint32(k)) & np.uint32(1)) << np.uint32(31 - k)
    np.testing.assert_array_equal(fx, exp)
    f = u32(q.radical_inverse_fill(n, 0))
    sel = np.random.default_rng(0).integers(0, n, 20000)
    np.testing.assert_array_equal(f[sel], mapv(exp[sel]))


def test_vdc_vs_reference(ref):
    # 8-aligned firsts take the 256-bit kernel (k_vdc8, incl. ragged ends and
    # the 2^31 reduction / u32 wraps inside a launch), the others k_vdc
    for first, n in [(0, 4099), (2**31 - 7, 100), (2**32 - 50, 50), (123456789, 1000),
                     (2**31 - 8 * 4000, 70003), (2**32 - 8 * 5000, 80005), (2**33 + 8, 65541)]:
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first & 0xFFFFFFFF, n, 0, 0, 0, ptr(exp)) == 0
        np.testing.assert_array_equal(u32(q.radical_inverse_fill(n, 0, first=first, fixed=True)), exp)


# --------------------------------------------------------------- Halton
@pytest.mark.parametrize("mode", ["plain", "linear", "faure"])
def test_halton_vs_golden(golden_arrays, mode):
    exp = golden_arrays["radinv_" + mode]  # [16][4096]
    got = u32(q.halton_fill(4096, 16, scramble=mode, fixed=True))
    np.testing.assert_array_equal(got.T, exp)


def test_radical_big_indices(golden_arrays):
    idx = golden_arrays["radinv_big_idx"]
    for j in range(8):
        for k in range(0, idx.size, 64):
            got = u32(q.radical_inverse_fill(1, j, first=int(idx[k]), fixed=True))
            assert got[0] == golden_arrays["radinv_big"][j, k]


def test_tabled_halton_equals_linear(golden_arrays):
    """TabledHalton (radical.cpp:308-350) == linear-scrambled Halton."""
    got = u32(q.halton_fill(512, 32, first=1000, scramble="linear", fixed=True))
    np.testing.assert_array_equal(got, golden_arrays["tabled_halton32_from1000"])


def test_halton_many_dims_vs_oracle(oracle):
    dims = 100
    got = u32(q.halton_fill(300, dims, first=(1 << 32) - 150, fixed=True))
    for k in range(0, 300, 7):
        i = ((1 << 32) - 150 + k) & 0xFFFFFFFF
        for j in range(0, dims, 3):
            assert got[k, j] == oracle.qo_radical_inverse_fixed(i, j)


_MODE = {"plain": 0, "linear": 1, "faure": 2}


@pytest.mark.parametrize("pi", [1, 2, 3, 6, 17, 18, 40, 100, 563, 564, 999])
@pytest.mark.parametrize("mode", ["plain", "linear", "faure"])
def test_radical_fill_windows_vs_reference(ref, pi, mode):
    """Contiguous fills (incremental hi/lo split, table bases up to 4096, the
    per-sample loop beyond) against the reference per index: windows across
    prime_max_power (i %= maxpow), across 2^31 and across the u32 wrap."""
    b, mp = q.prime(pi), q.prime_max_power(pi)
    factor = max(1, (b * 5) // 7) if mode == "linear" else 1
    for first, n in [(0, 5000), (mp - 2100, 4200), (2**31 - 1000, 3000), (2**32 - 2000, 3000),
                     (987654321, 3000), (3 * mp + 17, 777)]:
        if first + n > 2**32 + 2000:
            continue
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first & 0xFFFFFFFF, n, pi, _MODE[mode], factor,
                                          ptr(exp)) == 0
        got = u32(q.radical_inverse_fill(n, pi, first=first, scramble=mode, factor=factor,
                                         fixed=True))
        np.testing.assert_array_equal(got, exp, err_msg=f"first={first}")


@pytest.mark.parametrize("mode", ["plain", "linear", "faure"])
def test_halton_fill_windows_vs_reference(ref, mode):
    dims = 40
    for first, n in [(0, 700), (3486784401 - 300, 700), (2**32 - 500, 700), (12345678, 333)]:
        got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
        for j in range(dims):
            b = q.prime(j)
            exp = np.zeros(n, np.uint32)
            assert ref.ref_radical_fixed_fill(first, n, j, _MODE[mode], b - 1 if b > 2 else 1,
                                              ptr(exp)) == 0
            np.testing.assert_array_equal(got[:, j], exp, err_msg=f"first={first} dim={j}")


@pytest.mark.parametrize("mode", ["plain", "faure"])
@pytest.mark.parametrize("first", [0, 3486784401 - (1 << 18), 2**32 - (1 << 18), 2**33 + 5])
def test_halton_fill_long_runs_vs_reference(ref, mode, first):
    """Long contiguous fills: the per-dimension state carried from tile to
    tile across the base-3 prime_max_power boundary and the u32 index wrap."""
    n, dims = 1 << 19, 12
    got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
    for j in range(dims):
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first & 0xFFFFFFFF, n, j, _MODE[mode], 1, ptr(exp)) == 0
        np.testing.assert_array_equal(got[:, j], exp, err_msg=f"dim={j}")


@pytest.mark.parametrize("dims", [1, 2, 3, 5, 8, 13, 16, 20, 31, 32])
def test_halton_fill_runs_all_small_dims_vs_reference(ref, dims):
    """dims <= 32 (k_halton_runs: runs x dims warps, state in registers):
    enough points for several sub-tiles per run on every SM, uneven runs, a
    ragged last sub-tile, and a start just below the base-3 prime_max_power."""
    n = 148 * 4 * 1500 + 777
    for first, mode in [(3486784401 - 100000, "linear"), (12345, "faure")]:
        got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
        for j in range(dims):
            b = q.prime(j)
            exp = np.zeros(n, np.uint32)
            assert ref.ref_radical_fixed_fill(first, n, j, _MODE[mode], b - 1 if b > 2 else 1,
                                              ptr(exp)) == 0
            np.testing.assert_array_equal(got[:, j], exp, err_msg=f"first={first} dim={j}")


def test_halton_fill_32_dims_small_and_ragged_vs_reference(ref):
    """dims == 32 (k_halton_tma: TMA boxes of 256 rows clipped at n) for
    counts below one box, one sub-tile and one CTA's share, u32 and f32."""
    for n, first in [(1, 0), (100, 7), (257, 2**32 - 100), (513, 1000), (148 * 512 + 33, 99)]:
        got = u32(q.halton_fill(n, 32, first=first, scramble="linear", fixed=True)).reshape(n, 32)
        f = q.halton_fill(n, 32, first=first, scramble="linear").cpu().numpy().reshape(n, 32)
        for j in range(32):
            b = q.prime(j)
            exp = np.zeros(n, np.uint32)
            assert ref.ref_radical_fixed_fill(first, n, j, 1, b - 1 if b > 2 else 1, ptr(exp)) == 0
            np.testing.assert_array_equal(got[:, j], exp, err_msg=f"n={n} dim={j}")
            mapped = np.zeros(n, np.uint32)
            ref.ref_map_bulk(ptr(exp), ptr(mapped), n)
            np.testing.assert_array_equal(f[:, j].view(np.uint32), mapped, err_msg=f"n={n} dim={j}")


@pytest.mark.parametrize("dims", [64, 96, 256, 36, 100, 300, 1000])
def test_halton_fill_column_blocks_vs_reference(ref, dims):
    """k_tma over 32-dimension column blocks (dims % 32 == 0, or dims % 4 == 0
    with a partial last block that the tensor store clips): a CTA's unit
    range crosses block boundaries, TMA boxes at column offset 32*cb."""
    n = 148 * 512 + 1000
    for first, mode in [(3486784401 - 20000, "linear"), (5, "faure")]:
        got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
        for j in list(range(0, dims, 5)) + [31, 32, dims - 1]:
            b = q.prime(j)
            exp = np.zeros(n, np.uint32)
            assert ref.ref_radical_fixed_fill(first, n, j, _MODE[mode], b - 1 if b > 2 else 1,
                                              ptr(exp)) == 0
            np.testing.assert_array_equal(got[:, j], exp, err_msg=f"first={first} dim={j}")


# ---------------------------------------------------------------- Sobol'
def test_sobol_vs_golden(golden_arrays, golden, oracle):
    got = u32(q.sobol_fill(1024, 64, fixed=True))
    np.testing.assert_array_equal(got, golden_arrays["sobol_fixed_1024x64"])
    f = q.sobol_fill(1 << 16, 32)
    assert fnv(oracle, u32(f)) == golden["sobol_f32_65536x32_fnv"]
    hi = golden_arrays["sobol_hi_idx"]
    for k in range(0, hi.size, 16):
        got = u32(q.sobol_fill(1, 64, first=int(hi[k]), fixed=True))
        np.testing.assert_array_equal(got.reshape(-1), golden_arrays["sobol_hi"][k])


@pytest.mark.parametrize("dims", [1, 2, 3, 4, 5, 8, 16, 32, 48, 64])
@pytest.mark.parametrize("first", [0, 77, 4096 * 3 + 5, (1 << 40) + 3, (1 << 52) - 3000])
def test_sobol_windows_vs_oracle(oracle, columns64, dims, first):
    n = 2500
    cols = np.ascontiguousarray(columns64[:dims])
    exp = np.zeros((n, dims), np.uint32)
    oracle.qo_sobol_fill_fixed(first, n, dims, ptr(cols), None, ptr(exp))
    got = u32(q.sobol_fill(n, dims, first=first, fixed=True)).reshape(n, dims)
    np.testing.assert_array_equal(got, exp)


def test_sobol_index_limit():
    with pytest.raises(ValueError):
        q.sobol_fill(10, 4, first=(1 << 52) - 5)
    with pytest.raises(q.ConfigError):
        q.sobol_fill(10, 65)  # builtin direction numbers provide 64 dims
    m = q.GeneratorMatrixSet.builtin(8)
    with pytest.raises(IndexError):
        q.sobol_fill(10, 9, matrices=m)


def test_sobol_xor_vs_golden(golden_arrays, golden, oracle):
    seeds = golden_arrays["seeds_c3"]
    f = q.sobol_fill(4096, 64, scramble="xor", words=seeds)
    assert fnv(oracle, u32(f)) == golden["sobol_xor_f32_4096x64_fnv"]


@pytest.mark.parametrize("dims", [1, 2, 3, 16, 32, 64])
def test_sobol_owen_vs_oracle(oracle, columns64, golden_arrays, mapv, dims):
    seeds = golden_arrays["seeds_c3"][:dims].copy()
    first, n = 1000, 3000
    cols = np.ascontiguousarray(columns64[:dims])
    exp = np.zeros((n, dims), np.uint32)
    oracle.qo_sobol_owen_fill_fixed(first, n, dims, ptr(cols), ptr(seeds), ptr(exp))
    got = u32(q.sobol_fill(n, dims, first=first, scramble="owen", words=seeds, fixed=True))
    np.testing.assert_array_equal(got.reshape(n, dims), exp)
    f = u32(q.sobol_fill(n, dims, first=first, scramble="owen", words=seeds))
    np.testing.assert_array_equal(f.reshape(n, dims)[::37], mapv(exp[::37]))


@pytest.mark.parametrize("dims", [3, 5, 7, 12, 24, 31, 33, 40, 62, 63, 99, 100, 96, 127, 160])
@pytest.mark.parametrize("scramble", ["none", "xor", "owen"])
def test_sobol_walk_dims_vs_oracle(oracle, columns64, dims, scramble):
    """One dimension per warp (k_runs for dims <= 32, k_tma column blocks for
    dims % 32 == 0) and, for wider rows, the slab kernel (k_sobol_slab):
    several sub-tiles per run, the 1024-index block steps, an unaligned first
    (head through the element-wise path), a ragged end."""
    rng = np.random.default_rng(dims)
    if dims <= 64:
        cols = np.ascontiguousarray(columns64[:dims])
        m = None
    else:
        cols = rng.integers(0, 2**32, (dims, 52), dtype=np.uint64).astype(np.uint32)
        m = q.GeneratorMatrixSet.from_columns(cols)
    words = [int(w) for w in rng.integers(0, 2**32, dims, dtype=np.uint64)]
    n = 148 * 1536 + 777
    for first in [0, 77, (1 << 40) + 3]:
        exp = np.zeros((n, dims), np.uint32)
        kw = {"matrices": m} if m is not None else {}
        if scramble == "owen":
            seeds = np.array(words, np.uint32)
            oracle.qo_sobol_owen_fill_fixed(first, n, dims, ptr(cols), ptr(seeds), ptr(exp))
            kw.update(scramble="owen", words=words)
        else:
            sw = np.array(words, np.uint32) if scramble == "xor" else None
            oracle.qo_sobol_fill_fixed(first, n, dims, ptr(cols), ptr(sw), ptr(exp))
            if scramble == "xor":
                kw.update(scramble="xor", words=words)
        got = u32(q.sobol_fill(n, dims, first=first, fixed=True, **kw)).reshape(n, dims)
        np.testing.assert_array_equal(got, exp, err_msg=f"first={first}")


@pytest.mark.parametrize("dims", [200, 700, 1000, 2500, 3000, 1001, 255, 1002])
@pytest.mark.parametrize("scramble", ["xor", "owen"])
def test_sobol_many_dims_vs_oracle(oracle, dims, scramble):
    """Direction-number sets with hundreds to thousands of dimensions: the
    slab kernel (4 or 8 dims per lane for dims % 4 == 0; 2 or 1 for the other
    widths above 128, k_sobol_slab<2|1>) and the 1024-thread tiled path."""
    rng = np.random.default_rng(dims)
    cols = rng.integers(0, 2**32, (dims, 52), dtype=np.uint64).astype(np.uint32)
    m = q.GeneratorMatrixSet.from_columns(cols)
    words = [int(w) for w in rng.integers(0, 2**32, dims, dtype=np.uint64)]
    n, first = 1500, 4096 * 5 + 77
    exp = np.zeros((n, dims), np.uint32)
    wa = np.array(words, np.uint32)
    if scramble == "owen":
        oracle.qo_sobol_owen_fill_fixed(first, n, dims, ptr(cols), ptr(wa), ptr(exp))
    else:
        oracle.qo_sobol_fill_fixed(first, n, dims, ptr(cols), ptr(wa), ptr(exp))
    got = u32(q.sobol_fill(n, dims, first=first, fixed=True, matrices=m, scramble=scramble,
                           words=words)).reshape(n, dims)
    np.testing.assert_array_equal(got, exp)


def test_max_dims_fills_vs_oracle(oracle):
    """The widest fills: Halton at the prime table's 1000 dims (shared-memory
    state for every dimension) and a 3000-dim lattice."""
    n, first = 700, 123457
    got = u32(q.halton_fill(n, 1000, first=first, fixed=True)).reshape(n, 1000)
    for j in (0, 1, 499, 998, 999):
        for k in (0, 1, 350, 699):
            assert got[k, j] == oracle.qo_radical_inverse_fixed(first + k, j)
    g = [2 * k + 1 for k in range(3000)]
    lat = u32(q.lattice_fill(n, g, first=first, fixed=True)).reshape(n, 3000)
    for j in (0, 1777, 2999):
        for k in (0, 699):
            assert lat[k, j] == oracle.qo_lattice_component_fixed(first + k, g[j])


# --------------------------------------------------------------- lattice
def test_lattice_vs_golden(golden_arrays, golden, oracle):
    g = golden_arrays["lfsr_ace1_16"]
    got = u32(q.lattice_fill(4096, g))
    np.testing.assert_array_equal(got, golden_arrays["lattice_f32_4096x16"].view(np.uint32))
    s = golden_arrays["cp_shifts16"]
    f = q.lattice_fill(1 << 16, g, first=(1 << 32) - 30000, shifts=s)
    assert fnv(oracle, u32(f)) == golden["lattice_cp_f32_wrap_fnv"]


@pytest.mark.parametrize("dims", [1, 2, 3, 4, 8, 16, 32, 64, 128, 96, 100, 200, 1000, 3000])
def test_lattice_dims_vs_oracle(oracle, dims):
    """Fast tiles (dims dividing 256 / 128), narrow kernels, and the wide-row
    slab kernel (dims > 64 otherwise, k_lattice_slab) across the 2^32 wrap."""
    rng = np.random.default_rng(dims)
    g = (rng.integers(0, 1 << 31, dims) * 2 + 1).astype(np.uint32)
    s = rng.integers(0, 1 << 32, dims, dtype=np.uint64).astype(np.uint32)
    first, n = (1 << 32) - 1000, 2100
    got = u32(q.lattice_fill(n, g, first=first, shifts=s, fixed=True)).reshape(n, dims)
    cols = range(dims) if dims <= 200 else sorted(set(range(0, dims, 37)) | {dims - 1})
    for k in range(0, n, 13):
        i = (first + k) & 0xFFFFFFFF
        for j in cols:
            assert got[k, j] == oracle.qo_lattice_cp_fixed(i, int(g[j]), int(s[j]))
    # float output of the same points: the bit-exact map of the integers
    f = q.lattice_fill(n, g, first=first, shifts=s).cpu().numpy().reshape(n, dims)
    for k in (0, 999, 1000, n - 1):
        for j in cols:
            assert f.view(np.uint32)[k, j] == oracle.qo_map_bits(int(got[k, j]))


# ------------------------------------------------------- stream façade
STREAM_CASES = [
    ("sobol", {}, 2, 256),
    ("halton", {}, 2, 256),
    ("lattice", {}, 2, 256),
    ("halton-hilbert", {"pixel": (3, 5), "order": 4, "spp": 16}, 2, 16),
    ("pixel-shifted-lattice", {"pixel": (3, 5), "order": 12}, 2, 256),
    ("pixel-random-lattice", {"pixel": (3, 5)}, 2, 256),
    ("image-plane-halton", {"pixel": (3, 5), "width": 64, "height": 64}, 6, 256),
]


@pytest.mark.parametrize("kind,extra,dims,n", STREAM_CASES)
def test_stream_vs_golden(golden_arrays, kind, extra, dims, n):
    kw = dict(extra)
    if kind in ("lattice", "pixel-shifted-lattice"):
        kw["generator"] = q.lfsr_generator_vector(0xACE1, max(dims, 2))
    got = u32(q.stream_fill(kind, n, dims, **kw))
    np.testing.assert_array_equal(got.reshape(n, dims),
                                  golden_arrays["stream_" + kind.replace("-", "_")])


@pytest.mark.parametrize("kind", ["pixel-shifted-lattice", "pixel-random-lattice",
                                  "image-plane-halton", "halton-hilbert", "sobol-xor-table"])
def test_stream_pixels_vs_reference(ref, kind):
    rng = np.random.default_rng(9)
    for _ in range(6):
        w, h = 3840, 2160
        px, py = int(rng.integers(0, w)), int(rng.integers(0, h))
        dims = 5 if kind != "pixel-shifted-lattice" else 2
        n, spp, seed = 300, 300, 0
        kw = {"pixel": (px, py)}
        if kind == "pixel-shifted-lattice":
            kw.update(order=12, generator=q.lfsr_generator_vector(0xACE1, 2))
        if kind == "image-plane-halton":
            kw.update(width=w, height=h)
        if kind == "halton-hilbert":
            kw.update(order=12, spp=spp)
        if kind == "sobol-xor-table":
            seed = 77
            kw.update(xor_seed=seed, xor_point_count=512, pixel=(px % 128, py % 128))
            px, py = px % 128, py % 128
        got = u32(q.stream_fill(kind, n, dims, **kw)).reshape(n, dims)
        exp = np.zeros((n, dims), np.uint32)
        rc = ref.ref_stream_fill(kind.encode(), dims, seed, b"plain", px, py,
                                 kw.get("order", 1), spp, w if kind == "image-plane-halton" else 0,
                                 h if kind == "image-plane-halton" else 0, 0, n, ptr(exp))
        assert rc == 0, ref.ref_last_error()
        np.testing.assert_array_equal(got, exp)


def test_stream_config_errors():
    with pytest.raises(q.ConfigError):
        q.stream_fill("nope", 4)
    with pytest.raises(q.ConfigError):
        q.stream_fill("lattice", 4, 2, generator=[1, 2])  # even component
    with pytest.raises(q.ConfigError):
        q.stream_fill("pixel-shifted-lattice", 4, 2, generator=[1, 3], pixel=(4, 0), order=2)
    with pytest.raises(IndexError):
        q.stream_fill("halton-hilbert", 5, 2, spp=4, order=2)


# ----------------------------------------------------------------- render
RENDER_KINDS = ["pixel-shifted-lattice", "image-plane-halton", "sobol", "pixel-random-lattice",
                "lattice", "halton", "halton-hilbert"]


@pytest.mark.parametrize("kind", RENDER_KINDS)
@pytest.mark.parametrize("accum", ["kahan", "int"])
def test_render64_vs_golden(golden_arrays, kind, accum):
    exp = golden_arrays["render64_%s_%s" % (kind.replace("-", "_"), accum)]
    got = q.render(64, 64, 16, kind=kind, accum=accum).cpu().numpy()
    rel = np.abs(got.astype(np.float64) - exp) / np.maximum(np.abs(exp), 1e-30)
    assert rel.max() <= 1e-6, (kind, accum, rel.max())
    mism = int((got.view(np.uint32) != exp.view(np.uint32)).sum())
    print("%s/%s: %d of %d pixels differ in bits (max rel %.2e)" % (kind, accum, mism, exp.size,
                                                                   rel.max()))


def test_render_xor_table_vs_reference(ref):
    exp = np.zeros((48, 40), np.float32)
    assert ref.ref_render(40, 48, 8, b"sobol-xor-table", b"kahan", 5, 4, ptr(exp)) == 0
    got = q.render(40, 48, 8, kind="sobol-xor-table", seed=5).cpu().numpy()
    rel = np.abs(got.astype(np.float64) - exp) / np.maximum(np.abs(exp), 1e-30)
    assert rel.max() <= 1e-6


def test_render_bands_equal_full():
    full = q.render(96, 80, 4).cpu().numpy()
    bands = [q.render(96, 80, 4, rows=(r0, r1)).cpu().numpy()
             for r0, r1 in [(0, 17), (17, 40), (40, 80)]]
    np.testing.assert_array_equal(np.concatenate(bands), full)


@pytest.mark.parametrize("kind", q.SAMPLER_KINDS)
def test_render_ragged_columns_vs_reference(ref, kind):
    """spp >= 8 renders through k_render's column order (columns grouped by
    sine-quadrant parity, host::render_column_order) and its per-warp
    classification: a width that is no multiple of 32 and crosses quadrant
    boundaries mid-warp, int bit-identical, Kahan within 1e-6."""
    w, h, spp = 333, 77, 16
    for accum in ("int", "kahan"):
        exp = np.zeros((h, w), np.float32)
        assert ref.ref_render(w, h, spp, kind.encode(), accum.encode(), 0, 8, ptr(exp)) == 0
        got = q.render(w, h, spp, kind=kind, accum=accum).cpu().numpy()
        if accum == "int":
            np.testing.assert_array_equal(got, exp)
        else:
            rel = np.abs(got.astype(np.float64) - exp) / np.maximum(np.abs(exp), 1e-30)
            assert rel.max() <= 1e-6, rel.max()


def test_render_bands_equal_full_classified():
    """Row bands at spp >= 8 (the column-ordered kernel) tile the image."""
    full = q.render(333, 77, 16).cpu().numpy()
    bands = [q.render(333, 77, 16, rows=(r0, r1)).cpu().numpy()
             for r0, r1 in [(0, 5), (5, 40), (40, 77)]]
    np.testing.assert_array_equal(np.concatenate(bands), full)


def test_render_seeded_sobol_vs_reference(ref):
    exp = np.zeros((32, 32), np.float32)
    assert ref.ref_render(32, 32, 8, b"sobol", b"int", 99, 4, ptr(exp)) == 0
    got = q.render(32, 32, 8, kind="sobol", accum="int", seed=99).cpu().numpy()
    assert np.max(np.abs(got.astype(np.float64) - exp) / np.maximum(exp, 1e-30)) <= 1e-6


def test_render4k_golden_checksums(golden, oracle):
    """BASELINE C5 (3840x2160, pixel-shifted lattice): the FNV-1a of the GPU
    image equals the reference build's (tests/golden/make_golden.py) for
    1 spp Kahan, 16 spp Kahan and 64 spp int — bit for bit."""
    assert len(golden["render4k_psl_fnv"]) == 3
    for key, h in golden["render4k_psl_fnv"].items():
        spp, accum = key.split("/")
        img = q.render(3840, 2160, int(spp), accum=accum).cpu().numpy()
        got = fnv(oracle, img)
        print("render4k %s: %s (reference %s)" % (key, got, h))
        assert got == h, (key, got, h)


# BASELINE C5 at its stated size against the reference render run on this
# box (render.cpp:83-143 with workers = nproc; glibc sin, so run here, not
# from a fixture). spp 64/256 take the classified disc/quadrant/neumaier_add_big
# fast path (kernels_render.cu); halton-hilbert at 256 spp has block starts
# 4^12*256 > 2^32, i.e. the (uint32_t)(block_start_ + index) wrap
# (imageplane.cpp:378, :440-442), and phi3's 7+7+6-digit branch.
C5_CASES = [
    ("pixel-shifted-lattice", "kahan", 64),
    ("pixel-shifted-lattice", "kahan", 256),
    ("pixel-shifted-lattice", "int", 256),
    ("image-plane-halton", "kahan", 64),
    ("image-plane-halton", "kahan", 256),
    ("halton-hilbert", "kahan", 64),
    ("halton-hilbert", "int", 256),
]


@pytest.mark.slow
@pytest.mark.parametrize("kind,accum,spp", C5_CASES)
def test_render_4k_c5_vs_reference(ref, kind, accum, spp):
    """BASELINE C5 at 3840x2160, spp 64 and 256: every pixel within 1e-6
    relative of the reference render (north_star tolerance); the number of
    pixels whose bits differ is printed (CUDA sin vs glibc sin can move the
    last ulp of a sample)."""
    import os

    w, h = 3840, 2160
    exp = np.zeros((h, w), np.float32)
    assert ref.ref_render(w, h, spp, kind.encode(), accum.encode(), 0, os.cpu_count() or 1,
                          ptr(exp)) == 0
    got = q.render(w, h, spp, kind=kind, accum=accum).cpu().numpy()
    rel = np.abs(got.astype(np.float64) - exp) / np.maximum(np.abs(exp), 1e-30)
    mism = int((got.view(np.uint32) != exp.view(np.uint32)).sum())
    print("C5 4K %s/%s/spp%d: %d of %d pixels differ in bits, max rel %.2e"
          % (kind, accum, spp, mism, exp.size, rel.max()))
    assert np.isfinite(got).all()
    assert rel.max() <= 1e-6, (kind, accum, spp, rel.max(), mism)


def test_scene_value_vs_reference(ref):
    rng = np.random.default_rng(4)
    xy = rng.random((100000, 2))
    got = q.scene_value(xy)
    exp = np.array([ref.ref_scene_value(x, y) for x, y in xy[:20000]])
    err = np.abs(got[:20000] - exp)
    print("scene_value: %d of 20000 differ (device sin vs libm), max abs %.2e"
          % (int((got[:20000] != exp).sum()), err.max()))
    assert err.max() <= 4e-15  # a few ulp of values in [0, 1.25]


def test_sin_cw_matches_cuda_sin_bit_for_bit():
    """device.cuh sin_cw (the render's sine: CUDA's reduction and polynomials
    without the infinity / Payne-Hanek checks) equals CUDA's double sin on
    every argument: scene_value through qmc_scene_value against the same
    expression in torch float64 on the GPU (torch.sin is libdevice __nv_sin),
    one rounded op per torch call like the kernel's explicit _rn intrinsics."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    n = 1 << 22
    xy = torch.rand((n, 2), dtype=torch.float64, device="cuda", generator=g)
    xy[: n // 4] *= 2.0                                   # the render's range [0, 2)
    xy[n // 4: n // 2] = (xy[n // 4: n // 2] - 0.5) * 2e6  # large |arg|, below 2^31
    xy[-8:] = torch.tensor([[0.0, 0.25], [0.5, 1.0], [1.0 / 16, 3.0 / 16], [1e-300, -0.0],
                            [-1.5, 2.0], [7.0, -7.0], [85.0, 85.4], [0.125, 0.375]],
                           dtype=torch.float64)
    got = q.scene_value(xy)
    k = 25.132741228718345
    x, y = xy[:, 0], xy[:, 1]
    s = torch.sin(x * k) * torch.sin(y * k)
    v = (s + 1.0) * 0.5
    dx, dy = x - 0.5, y - 0.5
    inside = (dx * dx + dy * dy) < (0.3 * 0.3)
    exp = torch.where(inside, v + 0.25, v)
    bad = (got != exp).sum().item()
    assert bad == 0, bad


def test_concurrent_host_threads():
    """The C-ABI is reentrant: 8 host threads on their own streams run fills,
    streams and renders at once (first use of per-base tables included) and
    get exactly the single-threaded results."""
    import threading
    import torch

    def work(k):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            a = q.radical_inverse_fill(5000, 900 + k, first=123, fixed=True, stream=s.cuda_stream)
            b = q.halton_fill(3000, 24 + k, first=77 * k, scramble="faure", fixed=True,
                              stream=s.cuda_stream)
            c = q.sobol_fill(4000, 5 + k, first=1 << 33, scramble="owen", words=list(range(5 + k)),
                             fixed=True, stream=s.cuda_stream)
            d = q.render(48, 40, 8, kind=q.SAMPLER_KINDS[k % len(q.SAMPLER_KINDS)],
                         stream=s.cuda_stream)
        s.synchronize()
        return [x.cpu() for x in (a, b, c, d)]

    results = [None] * 8

    def run(k):
        results[k] = work(k)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for k in range(8):
        again = work(k)
        for x, y in zip(results[k], again):
            assert torch.equal(x, y), k


@pytest.mark.parametrize("wh", [(2, 3), (5, 2), (64, 27)])
def test_image_plane_halton_long_streams_vs_reference(ref, wh):
    """The phi_3 fast path (two 7-digit table steps below 3^14) and the digit
    loop above it: image-plane Halton streams whose y dimension
    phi_3(ipy0 + i * 2^a) runs through [0, 2^23) and past 3^14 = 4782969,
    against the reference stream bit for bit (fp32 bits)."""
    w, h = wh
    n, dims = 1 << 21, 3
    for px, py in [(0, 0), (w - 1, h - 1)]:
        got = u32(q.stream_fill("image-plane-halton", n, dims, width=w, height=h,
                                pixel=(px, py))).reshape(n, dims)
        exp = np.zeros((n, dims), np.uint32)
        assert ref.ref_stream_fill(b"image-plane-halton", dims, 0, b"plain", px, py, 1, 1, w, h,
                                   0, n, ptr(exp)) == 0, ref.ref_last_error()
        np.testing.assert_array_equal(got, exp)


def test_lattice_shifted_block_identity():
    """SPEC.md:354-362 / lattice.cpp:157-170: block k of 2^m lattice points is
    block 0 under the integer shift lattice_shift_fixed(k, m, g) — the CP-shift
    input of the fill reproduces the index-offset fill bit for bit."""
    g = q.lfsr_generator_vector(0xACE1, 16)
    for k, m in [(1, 10), (5, 12), (77, 16), (3, 20)]:
        direct = q.lattice_fill(1 << m, g, first=k << m, fixed=True)
        shifted = q.lattice_fill(1 << m, g, shifts=q.lattice_shift_fixed(k, m, g), fixed=True)
        assert torch.equal(direct, shifted), (k, m)


@pytest.mark.parametrize("kind", ["sobol", "lattice", "halton", "image-plane-halton"])
def test_integrate_partials_split_equals_whole(kind):
    """qmc_integrate_partials over any split of the chunk range, combined by
    reduce_deterministic in chunk order (kahan) or summed (int), is exactly
    qmc_integrate's estimate — the multi-GPU integrate's invariant."""
    n, dims = 4096 * 53 + 77, 5
    kw = {"generator": q.lfsr_generator_vector(0xACE1, dims)} if kind == "lattice" else {}
    if kind == "image-plane-halton":
        kw.update(width=64, height=27, pixel=(3, 4))
    chunks = (n + 4095) // 4096
    for accum in ("kahan", "int"):
        whole = q.integrate(kind, "product-sine", n, dims, accum, **kw)["estimate"]
        cuts = [0, 1, 17, 40, chunks]
        if accum == "kahan":
            vals = np.concatenate([q.integrate_partials(kind, "product-sine", n, dims, a, b,
                                                        accum, **kw)
                                   for a, b in zip(cuts, cuts[1:])])
            est = q.reduce_deterministic(np.arange(chunks)[::-1], vals[::-1]) / n
        else:
            tot = sum(q.integrate_partials(kind, "product-sine", n, dims, a, b, accum, **kw)
                      for a, b in zip(cuts, cuts[1:]))
            est = float(tot) / 4294967296.0 / n
        assert est == whole, (kind, accum)
    with pytest.raises(IndexError):
        q.integrate_partials(kind, "product-sine", n, dims, 3, chunks + 1, **kw)


def _nccl_world1_worker(rank, port, out_path):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2307_15584_b200.distributed import (integrate_distributed, render_distributed,
                                                   render_distributed_samples)

    a = render_distributed(96, 40, 8).cpu().numpy()
    b = render_distributed_samples(96, 40, 8).cpu().numpy()
    e1 = integrate_distributed("sobol", "product-sine", 4096 * 9 + 1, 4)
    e2 = integrate_distributed("sobol", "product-sine", 4096 * 9 + 1, 4, "int")
    np.savez(out_path, a=a, b=b, e=np.array([e1, e2]))
    dist.destroy_process_group()


def test_distributed_paths_on_nccl_world1(tmp_path):
    """The multi-GPU drivers on a real NCCL group (world size 1 on this box):
    device placement and collectives run, results equal the 1-GPU calls."""
    import socket

    import torch.multiprocessing as mp

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    out = str(tmp_path / "r.npz")
    mp.spawn(_nccl_world1_worker, args=(port, out), nprocs=1, join=True)
    r = np.load(out)
    np.testing.assert_array_equal(r["a"], q.render(96, 40, 8).cpu().numpy())
    np.testing.assert_array_equal(r["b"], q.render(96, 40, 8, accum="int").cpu().numpy())
    assert r["e"][0] == q.integrate("sobol", "product-sine", 4096 * 9 + 1, 4)["estimate"]
    assert r["e"][1] == q.integrate("sobol", "product-sine", 4096 * 9 + 1, 4, "int")["estimate"]


@pytest.mark.parametrize("kind", ["halton-hilbert", "image-plane-halton", "halton"])
def test_render_4k_halton_kinds_vs_reference(ref, kind):
    """4K renders of the Halton kinds against the reference render: every
    phi_3 path (two table steps below 3^14, 7 + 7 + 6 digits above — the
    halton-hilbert block indices reach 4^12 * spp) bit for bit in int mode."""
    import os

    w, h, spp = 3840, 2160, 2
    exp = np.zeros((h, w), np.float32)
    assert ref.ref_render(w, h, spp, kind.encode(), b"int", 0, os.cpu_count() or 1,
                          ptr(exp)) == 0
    got = q.render(w, h, spp, kind=kind, accum="int").cpu().numpy()
    np.testing.assert_array_equal(got, exp)


@pytest.mark.parametrize("world", [1, 2, 4, 8, 3])
def test_fill_shards_equal_single_fill(world):
    """SURVEY §4 plan item 5 with G logical shards: the multi-GPU partition
    (index_shard: contiguous index ranges, no collective) gives identical
    bytes to the single fill for every generator."""
    import torch

    from paper_2307_15584_b200.distributed import index_shard

    first, n = (1 << 33) + 7, 300001
    g = q.lfsr_generator_vector(0xACE1, 16)
    fills = {
        "sobol": lambda a, c: q.sobol_fill(c, 32, first=a, fixed=True),
        "owen": lambda a, c: q.sobol_fill(c, 64, first=a, scramble="owen",
                                          words=list(range(64)), fixed=True),
        "lattice": lambda a, c: q.lattice_fill(c, g, first=a, shifts=list(range(16)), fixed=True),
        "halton": lambda a, c: q.halton_fill(c, 24, first=a, scramble="faure", fixed=True),
    }
    for name, fill in fills.items():
        whole = fill(first, n)
        parts = [fill(*index_shard(first, n, world, r)) for r in range(world)]
        assert torch.equal(torch.cat(parts, 0), whole), (name, world)


def test_render_devices_bands_equal_one_device():
    """qmc_render_devices: row bands on a device list (here device 0 three
    times, one host thread each) assemble the one-device image bit for bit,
    into pinned and pageable host memory; errors as documented."""
    import torch

    for kind, accum in [("pixel-shifted-lattice", "kahan"), ("sobol", "int"),
                        ("image-plane-halton", "kahan")]:
        full = q.render(300, 77, 16, kind=kind, accum=accum).cpu().numpy()
        got = q.render_devices(300, 77, 16, [0, 0, 0], kind=kind, accum=accum)
        np.testing.assert_array_equal(got, full)
        pinned = torch.empty((77, 300), dtype=torch.float32, pin_memory=True).numpy()
        q.render_devices(300, 77, 16, [0] * 5, kind=kind, accum=accum, out=pinned)
        np.testing.assert_array_equal(pinned, full)
    with pytest.raises(ValueError):
        q.render_devices(300, 77, 16, [])
    with pytest.raises(ValueError):
        q.render_devices(300, 77, 16, [0], out=torch.empty((77, 300), device="cuda"))
    with pytest.raises(q.ConfigError):
        q.render_devices(300, 77, 0, [0, 0])


def test_render_samples_devices_fused_reduction():
    """qmc_render_samples_devices: parts k of n (the paper's sample partition)
    atomically add their int64 partials into one accumulator from their own
    kernels (here all on device 0; across GPUs through peer access) — the
    finalized image equals the one-device int render bit for bit."""
    for kind in ("pixel-shifted-lattice", "sobol", "image-plane-halton", "halton-hilbert"):
        full = q.render(200, 61, 24, kind=kind, accum="int").cpu().numpy()
        for n in (1, 2, 4, 8):
            got = q.render_samples_devices(200, 61, 24, [0] * n, kind=kind)
            np.testing.assert_array_equal(got, full, err_msg=f"{kind} n={n}")
    with pytest.raises(ValueError):
        q.render_samples_devices(200, 61, 24, [0, 0, 0])
    job_err = pytest.raises(ValueError)
    with job_err:
        q.render_samples_devices(200, 61, 24, [])


# ------------------------------------------------ full-size properties
@pytest.mark.slow
def test_c2_full_size_properties(oracle, columns64):
    """Config C2 (2^28 x 32) materialised: stratification of each dimension at
    m = 28, F2-linearity on random pairs, random rows vs the oracle."""
    n, dims = 1 << 28, 32
    x = q.sobol_fill(n, dims, fixed=True)  # 32 GiB
    rng = np.random.default_rng(1)
    rows = torch.from_numpy(rng.integers(0, n, 4096)).cuda()
    sample = u32(x[rows]).reshape(-1, dims)
    cols = np.ascontiguousarray(columns64[:dims])
    for k, i in enumerate(rows.cpu().tolist()):
        exp = np.zeros(dims, np.uint32)
        oracle.qo_sobol_fill_fixed(i, 1, dims, ptr(cols), None, ptr(exp))
        np.testing.assert_array_equal(sample[k], exp)
    a = torch.from_numpy(rng.integers(0, n, 1 << 20)).cuda()
    b = torch.from_numpy(rng.integers(0, n, 1 << 20)).cuda()
    np.testing.assert_array_equal(u32(x[a ^ b]), u32(x[a] ^ x[b]))  # x(a^b) = x(a)^x(b)
    for j in (0, 1, 7, 31):
        col = x[:, j].to(torch.int64) & 0xFFFFFFFF
        strata = torch.bincount(col >> 4, minlength=1 << 28)  # m = 28
        assert int(strata.min()) == 1 and int(strata.max()) == 1
        del col, strata
    del x
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("dims,n", [(48, 1 << 27), (12, 1 << 30), (24, (1 << 28) + 12345)])
def test_generic_dims_full_size(oracle, columns64, dims, n):
    """The element-wise Sobol' kernel (dims not dividing 256) and the Halton
    fill at tens of GiB (more than 2^32 output words): random rows against
    the oracle / the per-index reference, F2-linearity, and stratification
    of one dimension at m = log2(n) where n is a power of two."""
    x = q.sobol_fill(n, dims, first=7 if n & (n - 1) else 0, fixed=True)
    rng = np.random.default_rng(dims)
    rows = torch.from_numpy(rng.integers(0, n, 2048)).cuda()
    sample = u32(x[rows]).reshape(-1, dims)
    cols = np.ascontiguousarray(columns64[:dims])
    first = 7 if n & (n - 1) else 0
    for k, i in enumerate(rows.cpu().tolist()):
        exp = np.zeros(dims, np.uint32)
        oracle.qo_sobol_fill_fixed(first + i, 1, dims, ptr(cols), None, ptr(exp))
        np.testing.assert_array_equal(sample[k], exp)
    if first == 0:
        a = torch.from_numpy(rng.integers(0, n, 1 << 20)).cuda()
        b = torch.from_numpy(rng.integers(0, n, 1 << 20)).cuda()
        np.testing.assert_array_equal(u32(x[a ^ b]), u32(x[a] ^ x[b]))
        m = n.bit_length() - 1
        col = x[:, dims - 1].to(torch.int64) & 0xFFFFFFFF
        strata = torch.bincount(col >> (32 - m), minlength=1 << m)
        assert int(strata.min()) == 1 and int(strata.max()) == 1
        del col, strata
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dims", [8, 100, 128, 129, 200, 256, 300])
def test_large_dims_args_paths(oracle, dims):
    """Per-dim word arrays beyond the by-value parameter block (dims > 256)
    take the device-copy path; dims <= 128 not dividing 256 the element-wise
    kernel, larger ones the tiled kernel. XOR and Owen match the oracle."""
    rng = np.random.default_rng(dims)
    cols = rng.integers(0, 1 << 32, (dims, 52), dtype=np.uint64).astype(np.uint32)
    m = q.GeneratorMatrixSet.from_columns(cols)
    words = rng.integers(0, 1 << 32, dims, dtype=np.uint64).astype(np.uint32)
    n, first = 3000, (1 << 33) + 12345
    got = u32(q.sobol_fill(n, dims, first=first, scramble="xor", words=words, matrices=m,
                           fixed=True)).reshape(n, dims)
    exp = np.zeros((n, dims), np.uint32)
    oracle.qo_sobol_fill_fixed(first, n, dims, ptr(cols), ptr(words), ptr(exp))
    np.testing.assert_array_equal(got, exp)
    got = u32(q.sobol_fill(n, dims, first=first, scramble="owen", words=words, matrices=m,
                           fixed=True)).reshape(n, dims)
    oracle.qo_sobol_owen_fill_fixed(first, n, dims, ptr(cols), ptr(words), ptr(exp))
    np.testing.assert_array_equal(got, exp)
    g = (rng.integers(0, 1 << 31, dims) * 2 + 1).astype(np.uint32)
    s = rng.integers(0, 1 << 32, dims, dtype=np.uint64).astype(np.uint32)
    lat = u32(q.lattice_fill(n, g, first=first, shifts=s, fixed=True)).reshape(n, dims)
    for k in range(0, n, 61):
        for j in range(0, dims, 7):
            assert lat[k, j] == oracle.qo_lattice_cp_fixed(first + k, int(g[j]), int(s[j]))


def test_repeated_calls_stay_fast():
    """No per-call device allocation stalls: 10 back-to-back XOR fills of a
    2 GiB buffer (each ~0.35 ms, far above host-launch jitter) keep their
    device time within 2.5x of the median. The calls are queued without
    synchronising, so a stall inside a call shows up on the device timeline."""
    n, dims = 1 << 24, 32
    out = torch.empty((n, dims), dtype=torch.float32, device="cuda")
    words = list(range(1, dims + 1))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(12)]
    for a, b in ev:
        a.record()
        q.sobol_fill(n, dims, scramble="xor", words=words, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev[2:])
    assert ms[-1] < 2.5 * ms[len(ms) // 2], ms


def test_host_output_pipeline_matches_device():
    """HOST outputs (the e2e path: chunked device fill + D2H) equal the
    device fills, across many 64 MiB chunks, pinned and pageable."""
    n, dims = (1 << 21) + 77, 64  # ~512 MiB -> 9 chunks
    dev = u32(q.sobol_fill(n, dims, first=5, scramble="owen", words=list(range(64)), fixed=True))
    pinned = torch.empty((n, dims), dtype=torch.int32, pin_memory=True).numpy()
    q.sobol_fill(n, dims, first=5, scramble="owen", words=list(range(64)), fixed=True, out=pinned)
    np.testing.assert_array_equal(pinned.view(np.uint32), dev.reshape(n, dims))
    page = np.empty((3001, 16), np.float32)
    g = q.lfsr_generator_vector(0xACE1, 16)
    q.lattice_fill(3001, g, first=99, out=page)
    np.testing.assert_array_equal(page.view(np.uint32), u32(q.lattice_fill(3001, g, first=99)))
    img = np.empty((40, 64), np.float32)
    q.render(64, 64, 4, rows=(10, 50), out=img)
    np.testing.assert_array_equal(img, q.render(64, 64, 4, rows=(10, 50)).cpu().numpy())


def test_empty_and_degenerate_fills():
    out = torch.full((4, 4), 7.0, device="cuda")
    q.sobol_fill(0, 4, out=out)
    q.lattice_fill(0, [1, 3, 5, 7], out=out)
    q.halton_fill(0, 4, out=out)
    assert float(out.sum()) == 7.0 * 16  # nothing written
    one = u32(q.sobol_fill(1, 1, first=(1 << 52) - 1, fixed=True))
    assert one.size == 1


# ------------------------------------------------------------- integrate
def test_integrate_vs_reference_goldens(golden):
    """integrate() (quality.cpp:214-282) for every recorded (kind, integrand,
    accum, dims, n): same chunking and combine order as the reference; the
    estimate agrees to 1e-12 relative (FP64 sin is the only non-bit-exact
    step) and is reported bit-exact where it is."""
    exact = 0
    for kind, seed, f, accum, dims, n, est in golden["integrate"]:
        kw = {}
        if kind == "lattice":
            kw["generator"] = q.lfsr_generator_vector(0xACE1, max(dims, 2))
        if kind == "sobol" and seed:
            kw["sobol_scrambles"] = [q.pixel_hash(j, seed, 0x5EED) for j in range(dims)]
        row = q.integrate(kind, f, n, dims, accum, **kw)
        assert row["n"] == n
        rel = abs(row["estimate"] - est) / max(abs(est), 1e-300)
        assert rel <= 1e-12, (kind, seed, f, accum, dims, n, row["estimate"], est)
        exact += row["estimate"] == est
        _, ex = q.builtin_integrand(f, dims)
        assert row["abs_error"] == abs(row["estimate"] - ex)
    print("integrate: %d of %d estimates bit-identical to the reference"
          % (exact, len(golden["integrate"])))
    assert exact >= len(golden["integrate"]) // 2


def test_integrate_errors():
    with pytest.raises(ValueError):
        q.integrate("sobol", "product-sine", 0, 3)
    with pytest.raises(ValueError):
        q.integrate("sobol", "product-sine", 100, 3, stream_dims=2)
    with pytest.raises(q.ConfigError):
        q.integrate("sobol", "nope", 100, 3)
    with pytest.raises(ValueError):
        q.builtin_integrand("indicator", 0)
    assert q.builtin_integrand("indicator", 3)[1] == 0.7 ** 3


def test_integrate_pixel_kinds_vs_reference(ref):
    import ctypes as C
    for kind in ["halton", "pixel-random-lattice"]:
        for f in ["product-sine", "product-poly"]:
            e = C.c_double()
            assert ref.ref_integrate(kind.encode(), 4, 0, f.encode(), 50000, b"kahan", 4,
                                     C.byref(e)) == 0
            row = q.integrate(kind, f, 50000, 4)
            assert abs(row["estimate"] - e.value) <= 1e-12 * abs(e.value)


@pytest.mark.parametrize("accum", ["int", "kahan"])
def test_integrate_halton_quotient_tables_vs_reference(ref, accum):
    """Halton integration over 2^20 points x 12 dims: the chunks that take the
    quotient-table path (fill-table blocks h0, h0 + 1, incl. the ones that
    straddle a block) and the digit-loop fallback give the reference's
    estimate bit for bit (product-poly: exact FP64 products)."""
    import ctypes as C
    n, dims = (1 << 20) + 123, 12
    e = C.c_double()
    assert ref.ref_integrate(b"halton", dims, 0, b"product-poly", n, accum.encode(), 8,
                             C.byref(e)) == 0
    row = q.integrate("halton", "product-poly", n, dims, accum)
    assert row["estimate"] == e.value


@pytest.mark.parametrize("scramble", ["plain", "faure", "linear"])
@pytest.mark.parametrize("kind", ["halton", "halton-hilbert"])
def test_halton_streams_scrambles_vs_reference(ref, kind, scramble):
    dims, n = 7, 200
    kw = {"scramble": scramble}
    px = py = 0
    order, spp = 1, 1
    if kind == "halton-hilbert":
        px, py, order, spp = 5, 9, 5, n
        kw.update(pixel=(px, py), order=order, spp=spp)
    got = u32(q.stream_fill(kind, n, dims, **kw)).reshape(n, dims)
    exp = np.zeros((n, dims), np.uint32)
    assert ref.ref_stream_fill(kind.encode(), dims, 0, scramble.encode(), px, py, order, spp, 0,
                               0, 0, n, ptr(exp)) == 0, ref.ref_last_error()
    np.testing.assert_array_equal(got, exp)


def _strata_ok(col_i32, m):
    """Every one of the 2^m equal strata holds exactly one value."""
    v = (col_i32.to(torch.int64) & 0xFFFFFFFF) >> (32 - m)
    c = torch.bincount(v, minlength=1 << m)
    return int(c.min()) == 1 and int(c.max()) == 1


@pytest.mark.slow
def test_c3_owen_full_size_properties(oracle, columns64, golden_arrays):
    """Config C3 (Owen, 2^28 x 64) at full size: random rows equal the oracle
    and every dimension keeps one-point-per-stratum at m = 28 (Owen
    scrambling preserves the (0,m)-net property of each coordinate)."""
    n, dims = 1 << 28, 64
    seeds = golden_arrays["seeds_c3"]
    x = q.sobol_fill(n, dims, scramble="owen", words=seeds, fixed=True)  # 64 GiB
    rng = np.random.default_rng(3)
    rows = rng.integers(0, n, 2048)
    got = u32(x[torch.from_numpy(rows).cuda()]).reshape(-1, dims)
    exp = np.zeros((1, dims), np.uint32)
    for k, i in enumerate(rows.tolist()):
        oracle.qo_sobol_owen_fill_fixed(i, 1, dims, ptr(columns64), ptr(seeds), ptr(exp))
        np.testing.assert_array_equal(got[k], exp[0])
    for j in (0, 5, 33, 63):
        assert _strata_ok(x[:, j], 28), j
    del x
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_c4_lattice_cp_full_size_properties(oracle, golden_arrays):
    """Config C4 (2^30 x 16 + CP rotation) at full size: random rows equal
    the oracle; the first 2^26 points of every dimension are stratified at
    m = 26 (a shifted rank-1 lattice with odd g); the block identity
    x(i + k 2^m) = x(i) + Delta_k holds (lattice.cpp:157-170)."""
    n, dims = 1 << 30, 16
    g = golden_arrays["lfsr_ace1_16"]
    s = golden_arrays["cp_shifts16"]
    x = q.lattice_fill(n, g, shifts=s, fixed=True)  # 64 GiB
    rng = np.random.default_rng(4)
    rows = rng.integers(0, n, 2048)
    got = u32(x[torch.from_numpy(rows).cuda()]).reshape(-1, dims)
    for k, i in enumerate(rows.tolist()):
        for j in range(dims):
            assert got[k, j] == oracle.qo_lattice_cp_fixed(i, int(g[j]), int(s[j]))
    for j in range(0, dims, 5):
        assert _strata_ok(x[: 1 << 26, j], 26), j
    m, kk = 20, 37
    delta = np.zeros(dims, np.uint32)
    assert oracle.qo_lattice_shift_fixed(kk, m, ptr(g), dims, ptr(delta)) == 0
    a = u32(x[: 1 << 16]).astype(np.uint64)
    b = u32(x[kk << m: (kk << m) + (1 << 16)]).astype(np.uint64)
    np.testing.assert_array_equal(((a + delta[None, :]) & 0xFFFFFFFF).astype(np.uint32),
                                  b.astype(np.uint32))
    del x
    torch.cuda.empty_cache()


# --------------------------------------------------------- quality metrics
def test_quality_metrics_vs_reference(ref):
    import ctypes as C
    for dims, n in [(2, 4096), (5, 1000), (1, 17)]:
        pts = u32(q.sobol_fill(n, dims, first=3)).view(np.float32).reshape(n, dims).copy()
        e = C.c_double()
        assert ref.ref_l2_star(ptr(pts), n, dims, C.byref(e)) == 0
        got = q.l2_star_discrepancy(pts)
        assert abs(got - e.value) <= 1e-12 * e.value, (got, e.value)
        if n >= 2:
            assert ref.ref_min_toroidal(ptr(pts), n, dims, C.byref(e)) == 0
            assert q.min_toroidal_distance(torch.from_numpy(pts).cuda()) == e.value  # bit-exact
    one = np.zeros((1, 1), np.float32)
    assert abs(q.l2_star_discrepancy(one) - (1 / 3) ** 0.5) < 1e-15
    with pytest.raises(ValueError):
        q.min_toroidal_distance(one)


@pytest.mark.parametrize("kind,dims", [("sobol", 8), ("lattice", 4), ("halton", 3)])
def test_stratification_vs_reference(ref, kind, dims):
    import ctypes as C
    kw = {"generator": q.lfsr_generator_vector(0xACE1, max(dims, 2))} if kind == "lattice" else {}
    for j in range(dims):
        for m in (1, 8, 12, 20):
            ok, hist = q.check_1d_stratification(kind, j, m, dims, **kw)
            r = C.c_int()
            assert ref.ref_stratification(kind.encode(), dims, 0, j, m, C.byref(r)) == 0
            assert ok == bool(r.value), (kind, j, m)
            assert hist.sum() == 1 << m
    with pytest.raises(ValueError):
        q.check_1d_stratification("sobol", 0, 21, 2)


# ------------------------------------------------------------ XOR tables
def test_xor_tables_file_roundtrip_and_sampling(ref):
    """XQT1 tables: the reference writes a white-noise file; the product loads
    it with the CLI's stored point set and samples bit-identically; our
    writer reproduces the same bytes (imageplane.cpp:154-248)."""
    import ctypes as C
    dims, pc, seed = 3, 256, 9
    n = C.c_uint64(0)
    assert ref.ref_white_noise_xor_file(dims, pc, seed, None, C.byref(n)) == 0
    buf = np.zeros(n.value, np.uint8)
    assert ref.ref_white_noise_xor_file(dims, pc, seed, ptr(buf), C.byref(n)) == 0
    data = buf.tobytes()
    assert data[:4] == b"XQT1"
    # the product's white-noise tables write the same file
    assert q.XorTables.white_noise(dims, pc, seed).to_bytes() == data
    # CLI point set: Sobol' fixed points, XOR-scrambled with pixel_hash(j, seed, 0x5eed)
    words = [q.pixel_hash(j, seed, 0x5EED) for j in range(dims)]
    pts = u32(q.sobol_fill(pc, dims, scramble="xor", words=words, fixed=True)).reshape(pc, dims)
    t = q.XorTables.load(data, dims, pts, pc)
    assert (t.dims, t.point_count) == (dims, pc)
    for px, py in [(0, 0), (5, 77), (127, 127), (300, 129)]:
        got = u32(q.stream_fill("sobol-xor-table", pc, dims, xor_tables=t,
                                pixel=(px, py))).reshape(pc, dims)
        exp = np.zeros((pc, dims), np.uint32)
        assert ref.ref_xor_stream_fill(data, len(data), dims, seed, pc, px, py, 0, pc,
                                       ptr(exp)) == 0, ref.ref_last_error()
        np.testing.assert_array_equal(got, exp)
    with pytest.raises(q.ConfigError):
        q.XorTables.load(b"XQT0" + data[4:], dims, pts, pc)
    with pytest.raises(q.ConfigError):
        q.XorTables.load(data[:100], dims, pts, pc)
    with pytest.raises(IndexError):
        q.stream_fill("sobol-xor-table", pc + 1, dims, xor_tables=t)


def test_render_with_loaded_tables(ref):
    """render() with caller tables equals render() with the white-noise
    tables the job would build (render.cpp:102-104)."""
    spp, seed = 8, 4
    t = q.XorTables.white_noise(2, 8, seed)
    a = q.render(40, 30, spp, kind="sobol-xor-table", seed=seed).cpu().numpy()
    b = q.render(40, 30, spp, kind="sobol-xor-table", seed=seed, tables=t).cpu().numpy()
    np.testing.assert_array_equal(a, b)


def test_fills_capture_in_cuda_graph():
    """Fills are stream-ordered single launches with no host sync, so they
    can be captured in a CUDA graph and replayed (launch-bound configs)."""
    n = 1 << 16
    out = torch.zeros(n * 32, dtype=torch.float32, device="cuda")
    ref_out = q.sobol_fill(n, 32, first=7, scramble="xor", words=list(range(32)))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        q.sobol_fill(n, 32, first=7, scramble="xor", words=list(range(32)), out=out,
                     stream=s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(out), u32(ref_out).reshape(-1))


@pytest.mark.parametrize("kind", RENDER_KINDS + ["sobol-xor-table"])
def test_render_sample_partition_equals_int_render(kind):
    """The paper's sample partition on one GPU: the int64 partials of parts
    1, 2, 4, 8 (i == rev_2(part) mod parts) sum to exactly the int render."""
    w, h, spp = 48, 40, 24
    full = q.render(w, h, spp, kind=kind, accum="int", seed=3).cpu().numpy()
    for parts in (1, 2, 4, 8):
        acc = sum(q.render_partial(w, h, spp, part, parts, kind=kind, seed=3)
                  for part in range(parts))
        img = q.render_finalize(acc, spp).cpu().numpy()
        np.testing.assert_array_equal(img, full)
    with pytest.raises(q.ConfigError):
        q.render_partial(w, h, spp, 0, 3)
    with pytest.raises(IndexError):
        q.render_partial(w, h, spp, 4, 4)


# ---------------------------------------------- out-of-bounds write canaries
GUARD = 4096  # words of canary on each side (compute-sanitizer is closed on this pool)


def _guarded(n_words, dtype=torch.int32):
    buf = torch.full((n_words + 2 * GUARD,), 0x5A5A5A5A, dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + n_words]


def _canaries_intact(buf):
    head, tail = buf[:GUARD], buf[-GUARD:]
    return bool((head == 0x5A5A5A5A).all()) and bool((tail == 0x5A5A5A5A).all())


@pytest.mark.parametrize("dims", [1, 2, 3, 4, 8, 16, 32, 48, 64, 128, 256])
def test_fills_write_exactly_their_range(dims):
    for first, n in [(0, 1), (5, 777), (4096 * 7 + 3, 5000), ((1 << 40) + 11, 3001)]:
        for call in (
            lambda o: q.sobol_fill(n, dims, first=first, matrices=q.GeneratorMatrixSet.from_columns(
                np.arange(dims * 52, dtype=np.uint32).reshape(dims, 52) | 1), out=o),
            lambda o: q.sobol_fill(n, dims, first=first, scramble="owen", out=o,
                                   words=list(range(dims)),
                                   matrices=q.GeneratorMatrixSet.from_columns(
                                       np.arange(dims * 52, dtype=np.uint32).reshape(dims, 52))),
            lambda o: q.lattice_fill(n, [2 * k + 1 for k in range(dims)], first=first, out=o),
            lambda o: q.halton_fill(n, dims, first=first, out=o),
        ):
            buf, mid = _guarded(n * dims)
            call(mid)
            torch.cuda.synchronize()
            assert _canaries_intact(buf), (dims, first, n)


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_fills_misaligned_outputs(shift):
    """Outputs 4, 8 or 12 bytes off a 16-B boundary take the scalar store paths
    (no v4/v8 stores): same values as the aligned fill, canaries intact."""
    cases = [
        (8, lambda n, d, o: q.sobol_fill(n, d, first=77, fixed=True, out=o)),
        (32, lambda n, d, o: q.sobol_fill(n, d, scramble="owen", words=list(range(d)), fixed=True,
                                          out=o)),
        (16, lambda n, d, o: q.lattice_fill(n, q.lfsr_generator_vector(0xACE1, d), first=5,
                                            shifts=list(range(d)), fixed=True, out=o)),
        (32, lambda n, d, o: q.halton_fill(n, d, first=1000, scramble="linear", fixed=True, out=o)),
        (12, lambda n, d, o: q.halton_fill(n, d, first=3486784401 - 999, fixed=True, out=o)),
        (1, lambda n, d, o: q.radical_inverse_fill(n, 5, first=12345, fixed=True, out=o)),
    ]
    n = 6001
    for dims, call in cases:
        ref_out = torch.empty(n * dims, dtype=torch.int32, device="cuda")
        call(n, dims, ref_out)
        buf = torch.full((n * dims + 2 * GUARD,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
        mid = buf[GUARD + shift: GUARD + shift + n * dims]
        call(n, dims, mid)
        torch.cuda.synchronize()
        assert torch.equal(mid, ref_out), dims
        head, tail = buf[:GUARD + shift], buf[GUARD + shift + n * dims:]
        assert bool((head == 0x5A5A5A5A).all()) and bool((tail == 0x5A5A5A5A).all()), dims


def test_halton_level_table_fill_writes_exactly_its_range():
    """k_halton_lv with every CTA's three walker groups busy over several
    ring rounds and a partial last sub-tile: canaries intact, and the u32 and
    f32 outputs agree through the map."""
    n, dims = 148 * 128 * 3 * 5 + 77, 32
    for first in (0, 3486784401 - 50000, (1 << 32) - 60000):
        buf, mid = _guarded(n * dims)
        q.halton_fill(n, dims, first=first, scramble="linear", fixed=True, out=mid)
        torch.cuda.synchronize()
        assert _canaries_intact(buf), first
        f = q.halton_fill(n, dims, first=first, scramble="linear")
        np.testing.assert_array_equal(
            f.cpu().numpy().view(np.uint32).ravel(),
            q.map_u32_to_unifloat(mid.view(torch.int32)).cpu().numpy().view(np.uint32).ravel())


def test_render_tables_and_host_bands_write_exactly_their_range():
    """spp >= 32 renders of the Halton kinds (phi_3 tables bulk-copied per
    CTA, halton-hilbert's record split) and a host image above 2^20 pixels
    (row bands, D2H overlapped) write only their rows: canaries intact."""
    for kind in ("image-plane-halton", "halton", "halton-hilbert"):
        buf, mid = _guarded(50 * 96)
        q.render(96, 80, 64, kind=kind, rows=(13, 63), out=mid.view(torch.float32))
        torch.cuda.synchronize()
        assert _canaries_intact(buf), kind
    rows, w = (3, 1103), 1000
    host = np.full((rows[1] - rows[0]) * w + 2 * GUARD, 0x5A5A5A5A, np.uint32)
    q.render(w, 1110, 4, rows=rows, out=host[GUARD:-GUARD].view(np.float32).reshape(-1, w))
    assert (host[:GUARD] == 0x5A5A5A5A).all() and (host[-GUARD:] == 0x5A5A5A5A).all()
    dev = q.render(w, 1110, 4, rows=rows).cpu().numpy()
    np.testing.assert_array_equal(host[GUARD:-GUARD], dev.view(np.uint32).ravel())


def test_render_and_streams_write_exactly_their_range():
    for kind in q.SAMPLER_KINDS:
        buf, mid = _guarded(23 * 37)
        q.render(37, 30, 3, kind=kind, rows=(4, 27), out=mid.view(torch.float32))
        torch.cuda.synchronize()
        assert _canaries_intact(buf), kind
        kw = {}
        if kind in ("lattice", "pixel-shifted-lattice"):
            kw["generator"] = q.lfsr_generator_vector(0xACE1, 3)
        if kind in ("halton-hilbert", "pixel-shifted-lattice"):
            kw.update(order=6, pixel=(5, 7))
        if kind == "halton-hilbert":
            kw["spp"] = 50
        if kind == "image-plane-halton":
            kw.update(width=30, height=20, pixel=(5, 7))
        if kind == "sobol-xor-table":
            kw.update(xor_point_count=64, xor_seed=3)
        buf, mid = _guarded(50 * 3)
        q.stream_fill(kind, 50, 3, out=mid, **kw)
        torch.cuda.synchronize()
        assert _canaries_intact(buf), kind


@pytest.mark.parametrize("kind", ["pixel-shifted-lattice", "sobol", "image-plane-halton",
                                  "pixel-random-lattice"])
def test_render_small_image_high_spp_warp_path(ref, kind):
    """Few pixels x many samples takes the warp-per-pixel kernel (shuffle
    reductions): int mode stays bit-identical to the reference's sequential
    int sum; Kahan mode within 1e-12 relative."""
    w, h, spp = 24, 16, 1000
    for accum in ("int", "kahan"):
        exp = np.zeros((h, w), np.float32)
        assert ref.ref_render(w, h, spp, kind.encode(), accum.encode(), 0, 8, ptr(exp)) == 0
        got = q.render(w, h, spp, kind=kind, accum=accum).cpu().numpy()
        if accum == "int":
            np.testing.assert_array_equal(got, exp)
        else:
            rel = np.abs(got.astype(np.float64) - exp) / np.maximum(np.abs(exp), 1e-30)
            assert rel.max() <= 1e-6, rel.max()


def test_write_pnm_matches_reference(ref):
    """write_pgm / write_ppm (image.cpp:25-52) of a render: byte-identical."""
    import ctypes as C
    img = q.render(57, 31, 8, kind="image-plane-halton")
    host = img.cpu().numpy()
    host[0, :4] = [-0.5, 1.5, 0.5, 0.998]  # clamp and rounding edges
    for ch, p6 in ((1, 0), (3, 1)):
        n = C.c_uint64(0)
        assert ref.ref_write_pnm(ptr(host), 57, 31, p6, None, C.byref(n)) == 0
        buf = np.zeros(n.value, np.uint8)
        assert ref.ref_write_pnm(ptr(host), 57, 31, p6, ptr(buf), C.byref(n)) == 0
        assert q.write_pnm(host, ch) == buf.tobytes()
        assert q.write_pnm(torch.from_numpy(host).cuda(), ch) == buf.tobytes()


# ------------------------------------------ the collective inside the library
def test_render_nccl_devices_world1_equals_render():
    """qmc_render_nccl_devices on a one-GPU NCCL communicator
    (ncclCommInitAll): row bands + ncclAllGather and the sample partition +
    int64 ncclAllReduce reproduce the one-GPU render bit for bit."""
    for kind in ("pixel-shifted-lattice", "image-plane-halton", "sobol"):
        full = q.render(300, 77, 16, kind=kind).cpu().numpy()
        np.testing.assert_array_equal(q.render_nccl_devices(300, 77, 16, [0], kind=kind), full)
        ifull = q.render(300, 77, 16, kind=kind, accum="int").cpu().numpy()
        got = q.render_nccl_devices(300, 77, 16, [0], mode="samples", kind=kind, accum="int")
        np.testing.assert_array_equal(got, ifull)
    with pytest.raises(ValueError):  # sample partitions need the int accumulator
        q.render_nccl_devices(300, 77, 16, [0], mode="samples")
    with pytest.raises(ValueError):
        q.render_nccl_devices(300, 77, 16, [])


def _comm_world1_worker(rank, port, out_path):
    import torch

    torch.cuda.set_device(0)
    comm = q.Comm.init_rank(q.Comm.unique_id(), 1, 0)
    info = comm.info()
    a = q.render_nccl(3840, 2160, 4, comm).cpu().numpy()
    b = q.render_nccl(3840, 2160, 4, comm, mode="samples", accum="int").cpu().numpy()
    c = q.render_nccl(97, 31, 9, comm, kind="halton-hilbert").cpu().numpy()
    comm.destroy()
    np.savez(out_path, a=a, b=b, c=c, info=np.array([info["rank"], info["nranks"],
                                                     info["device"]]))


def test_render_nccl_comm_init_rank_world1(tmp_path):
    """qmc_comm_unique_id + qmc_comm_init_rank + qmc_render_nccl in a fresh
    process (the torchrun shape at world size 1): the 4K image equals the
    one-GPU render bit for bit in both partition modes."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "c.npz")
    mp.spawn(_comm_world1_worker, args=(0, out), nprocs=1, join=True)
    r = np.load(out)
    assert list(r["info"]) == [0, 1, 0]
    np.testing.assert_array_equal(r["a"], q.render(3840, 2160, 4).cpu().numpy())
    np.testing.assert_array_equal(r["b"], q.render(3840, 2160, 4, accum="int").cpu().numpy())
    np.testing.assert_array_equal(r["c"], q.render(97, 31, 9, kind="halton-hilbert").cpu().numpy())


def _two_gpus():
    import torch

    return torch.cuda.device_count() >= 2


@pytest.mark.skipif(not _two_gpus(), reason="needs >= 2 GPUs")
def test_multi_gpu_renders_distinct_devices_4k():
    """Distinct GPUs: the peer-atomic sample partition, the row
    bands and the NCCL paths at 4K against the one-device render, including
    a device count that does not divide the height (scratch all-gather)."""
    import torch

    n = torch.cuda.device_count()
    devs = list(range(min(n, 8)))
    pow2 = devs[: 1 << (len(devs).bit_length() - 1)]
    full = q.render(3840, 2160, 8).cpu().numpy()
    ifull = q.render(3840, 2160, 8, accum="int").cpu().numpy()
    np.testing.assert_array_equal(q.render_devices(3840, 2160, 8, devs), full)
    np.testing.assert_array_equal(q.render_samples_devices(3840, 2160, 8, pow2), ifull)
    np.testing.assert_array_equal(q.render_nccl_devices(3840, 2160, 8, devs), full)
    np.testing.assert_array_equal(
        q.render_nccl_devices(3840, 2160, 8, pow2, mode="samples", accum="int"), ifull)
    odd = q.render(3840, 2161, 8).cpu().numpy()
    np.testing.assert_array_equal(q.render_nccl_devices(3840, 2161, 8, devs[:3] or devs), odd)


# ------------------------------- run_bench_kernel (SPEC acceptance 9's walk)
BENCH_KERNELS = ["sobol", "halton", "halton-tabled", "lattice", "pixel-shifted-lattice",
                 "pixel-random-lattice"]


@pytest.mark.parametrize("kernel", BENCH_KERNELS)
def test_bench_kernel_checksums_vs_golden(golden, kernel):
    """qmc_run_bench_kernel folds the same components in the same walk into
    the same Sink checksum as the reference's run_bench_kernel
    (bench.cpp:23-150): 65536 evaluations x 32 dims, golden from the
    reference build."""
    r = q.run_bench_kernel(kernel, 65536, 32)
    assert "%016x" % r["checksum"] == golden["bench_checksums_65536x32"][kernel]
    assert r["evaluations"] == 65536 and r["seconds"] > 0


@pytest.mark.parametrize("kernel", BENCH_KERNELS)
@pytest.mark.parametrize("count,dims", [(1, 1), (1000003, 7), (2621440, 32), (300001, 100)])
def test_bench_kernel_vs_reference(ref, kernel, count, dims):
    """Ragged counts (a partial last index), other dims and walks past one
    128x128 tile (py wraps) against the reference build's checksum."""
    import ctypes as C

    if kernel == "sobol" and dims > 64:
        with pytest.raises(q.ConfigError):
            q.run_bench_kernel(kernel, count, dims)
        return
    cps, ck = C.c_double(), C.c_uint64()
    assert ref.ref_run_bench_kernel(kernel.encode(), count, dims, C.byref(cps), C.byref(ck)) == 0
    assert q.run_bench_kernel(kernel, count, dims)["checksum"] == ck.value


def test_bench_kernel_errors():
    with pytest.raises(q.ConfigError):
        q.run_bench_kernel("nope", 10, 2)
    with pytest.raises(q.ConfigError):
        q.run_bench_kernel("lattice", 0, 2)
    with pytest.raises(q.ConfigError):
        q.run_bench_kernel("lattice", 10, 0)


def test_fp64_probe_reports_a_plausible_peak():
    tf = q.fp64_probe(2048) / 1e12
    print("fp64 probe: %.2f TFLOP/s" % tf)
    assert 5.0 < tf < 200.0


# --------------------------------------------- integrate beyond 64 dimensions
@pytest.mark.parametrize("kind,dims,integrand,accum", [
    ("halton", 100, "product-poly", "kahan"),
    ("halton", 100, "product-poly", "int"),
    ("halton", 500, "product-poly", "kahan"),
    ("halton", 500, "indicator", "int"),
    ("lattice", 200, "product-poly", "kahan"),
    ("lattice", 200, "indicator", "int"),
])
def test_integrate_high_dims_vs_reference(ref, kind, dims, integrand, accum):
    """integrate() (quality.cpp:214-282) has no dimension cap: Halton at 100
    and 500 dims (the first 64 dims on the quotient-table state, the rest on
    the digit loop) and lattice at 200 dims equal the reference bit for bit."""
    import ctypes as C

    n = 3 * 4096 + 77
    e = C.c_double()
    assert ref.ref_integrate(kind.encode(), dims, 0, integrand.encode(), n, accum.encode(), 8,
                             C.byref(e)) == 0
    kw = {"generator": q.lfsr_generator_vector(0xACE1, dims)} if kind == "lattice" else {}
    row = q.integrate(kind, integrand, n, dims, accum, **kw)
    assert row["estimate"] == e.value, (row["estimate"], e.value)


def _direction_text(dims, seed=5):
    """A valid direction-number file (the builtin 63 Joe-Kuo rows, then
    synthetic rows obeying parse_direction_numbers' grammar)."""
    import json

    rows = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))[
        "direction_numbers"]
    rng = np.random.default_rng(seed)
    lines = ["d s a m_i"]
    for d in range(2, dims + 1):
        if d - 2 < len(rows):
            _, s, a, ms = rows[d - 2]
        else:
            s = int(rng.integers(3, 12))
            a = int(rng.integers(0, 1 << (s - 1)))
            ms = [int(rng.integers(0, 1 << (k - 1))) * 2 + 1 for k in range(1, s + 1)]
        lines.append(" ".join(str(v) for v in [d, s, a] + list(ms)))
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("accum", ["kahan", "int"])
def test_integrate_sobol_beyond_64_dims_vs_reference(ref, accum):
    """Sobol' integration over caller direction numbers with 130 dims: the
    first 64 on the incremental state, the rest XOR the columns per sample —
    bit for bit with the reference."""
    import ctypes as C

    dims, n = 130, 2 * 4096 + 5
    text = _direction_text(dims)
    e = C.c_double()
    assert ref.ref_integrate_sobol_text(text.encode(), dims, b"product-poly", n, accum.encode(), 8,
                                        C.byref(e)) == 0, ref.ref_last_error()
    m = q.GeneratorMatrixSet.from_text(text, dims)
    row = q.integrate("sobol", "product-poly", n, dims, accum, matrices=m)
    assert row["estimate"] == e.value, (row["estimate"], e.value)


@pytest.mark.parametrize("dims", [1, 2, 3, 16, 32, 64, 300])
@pytest.mark.parametrize("first", [0, (1 << 32) - 5000, (1 << 33) + 17])
def test_pixel_shifted_lattice_stream_as_cp_lattice_vs_reference(ref, dims, first):
    """The pixel-shifted lattice stream goes through the lattice fill with
    integer shifts s_j = shift * g_j ((brev(i) + shift) * g_j mod 2^32,
    imageplane.hpp:26-31): every dims path (fast 256-bit, generic, > 256 dims
    device args), windows across the u32 index wrap, fixed and float — equal
    to SampleStream::sample of the reference."""
    px, py, order, n = 3001, 1777, 12, 9000
    g = q.lfsr_generator_vector(0xACE1, max(dims, 2))
    got = u32(q.stream_fill("pixel-shifted-lattice", n, dims, first=first, generator=g,
                            pixel=(px, py), order=order)).reshape(n, dims)
    exp = np.zeros((n, dims), np.uint32)
    assert ref.ref_stream_fill(b"pixel-shifted-lattice", dims, 0, b"plain", px, py, order, 1, 0, 0,
                               first, n, ptr(exp)) == 0, ref.ref_last_error()
    np.testing.assert_array_equal(got, exp)
    fx = u32(q.stream_fill("pixel-shifted-lattice", n, dims, first=first, generator=g,
                           pixel=(px, py), order=order, fixed=True)).reshape(n, dims)
    shift = q.hilbert_phi3_fixed(px, py, order)
    i = (np.arange(first, first + n, dtype=np.uint64) & 0xFFFFFFFF).astype(np.uint32)
    br = np.array([int("{:032b}".format(int(v))[::-1], 2) for v in i], np.uint64)
    ga = np.array(g[:dims], np.uint64)
    np.testing.assert_array_equal(
        fx, (((br[:, None] + shift) & 0xFFFFFFFF) * ga[None, :] & 0xFFFFFFFF).astype(np.uint32))


@pytest.mark.parametrize("mode", ["plain", "linear", "faure"])
@pytest.mark.parametrize("first", [0, 3486784401 - (1 << 18), 2**31 - (1 << 18) - 3,
                                   2**32 - (1 << 18) + 5, 2**33 + 5])
def test_halton_fill_q4_long_runs_vs_reference(ref, mode, first):
    """k_halton_q4 (dims % 32 == 0): 2^19 + 77 points x 32 dims carried
    across sub-tiles, across the base-3 prime_max_power boundary, the base-2
    2^31 reduction and the u32 index wrap (the per-sample fallback units)."""
    n, dims = (1 << 19) + 77, 32
    got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
    for j in range(dims):
        b = q.prime(j)
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first & 0xFFFFFFFF, n, j, _MODE[mode],
                                          b - 1 if (mode == "linear" and b > 2) else 1,
                                          ptr(exp)) == 0
        np.testing.assert_array_equal(got[:, j], exp, err_msg=f"dim={j}")


@pytest.mark.parametrize("kind", ["pixel-shifted-lattice", "image-plane-halton"])
def test_render_host_image_bands_equal_device(kind):
    """qmc_render into host memory renders in row bands whose D2H copies
    overlap the next band's render (>= 2^20 pixels): the host image equals
    the device render bit for bit, for the whole image and for a row range
    that does not split evenly into the bands."""
    import numpy as np
    for rows in [(0, 2160), (7, 2001)]:
        dev = q.render(3840, 2160, 16, kind=kind, rows=rows).cpu().numpy()
        host = np.empty_like(dev)
        q.render(3840, 2160, 16, kind=kind, rows=rows, out=host)
        np.testing.assert_array_equal(host.view(np.uint32), dev.view(np.uint32))


@pytest.mark.parametrize("mode", ["linear", "faure"])
@pytest.mark.parametrize("first", [3486784401 - (1 << 22) + 5, 2**32 - (1 << 22) - 77])
def test_halton_fill_level_tables_long_vs_reference(ref, mode, first):
    """k_halton_lv (dims == 32, on-chip level tables): 2^23 + 333 points, so
    every walker group crosses many G0 * G1 record blocks (record rebuilds
    from the shared q0 table), the base-3 prime_max_power reduction, the
    base-2 2^31 reduction, and the u32 index wrap (the per-sample sub-tile
    and the re-initialised walk after it), u32 and f32 outputs."""
    n, dims = (1 << 23) + 333, 32
    got = u32(q.halton_fill(n, dims, first=first, scramble=mode, fixed=True)).reshape(n, dims)
    f = q.halton_fill(n, dims, first=first, scramble=mode).cpu().numpy().reshape(n, dims)
    for j in range(dims):
        b = q.prime(j)
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first & 0xFFFFFFFF, n, j, _MODE[mode],
                                          b - 1 if (mode == "linear" and b > 2) else 1,
                                          ptr(exp)) == 0
        np.testing.assert_array_equal(got[:, j], exp, err_msg=f"dim={j}")
        mapped = np.zeros(n, np.uint32)
        ref.ref_map_bulk(ptr(exp), ptr(mapped), n)
        np.testing.assert_array_equal(f[:, j].view(np.uint32), mapped, err_msg=f"f32 dim={j}")


@pytest.mark.parametrize("dims", [64, 160])
def test_halton_fill_q4_many_blocks_vs_reference(ref, dims):
    """Column blocks past the first (bases up to 941 at 160 dims, fill tables
    of one or two digits with G >= 257): every dimension against the
    reference, f32 output through the map."""
    n, first = 40000 + 3, 123456789
    got = q.halton_fill(n, dims, first=first, scramble="linear").cpu().numpy().reshape(n, dims)
    for j in range(dims):
        b = q.prime(j)
        exp = np.zeros(n, np.uint32)
        assert ref.ref_radical_fixed_fill(first, n, j, 1, b - 1 if b > 2 else 1, ptr(exp)) == 0
        mapped = np.zeros(n, np.uint32)
        ref.ref_map_bulk(ptr(exp), ptr(mapped), n)
        np.testing.assert_array_equal(got[:, j].view(np.uint32), mapped, err_msg=f"dim={j}")


@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("first", [77, 4 * 1000 + 2, (1 << 33) + 17, (1 << 32) - 70001])
def test_narrow_fills_unaligned_first_vs_oracle(oracle, columns64, dims, first):
    """dims 1 and 2 over several 8192-point tiles from a first index that is
    not a multiple of 8 / dims (the narrow kernels' interior tiles use 32-B
    stores at out + (i - first) * dims): Sobol' (plain, XOR, Owen) and the
    CP lattice against the oracle."""
    n = 70001
    for sc in ("none", "xor", "owen"):
        words = [0x9E3779B9 * (j + 1) & 0xFFFFFFFF for j in range(dims)] if sc != "none" else None
        got = u32(q.sobol_fill(n, dims, first=first, scramble=sc, words=words, fixed=True))
        exp = np.zeros((n, dims), np.uint32)
        w = np.ascontiguousarray(words if words else [0] * dims, np.uint32)
        cols = np.ascontiguousarray(columns64[:dims])
        if sc == "owen":
            oracle.qo_sobol_owen_fill_fixed(first, n, dims, ptr(cols), ptr(w), ptr(exp))
        else:
            oracle.qo_sobol_fill_fixed(first, n, dims, ptr(cols), ptr(w) if words else None,
                                       ptr(exp))
        np.testing.assert_array_equal(got.reshape(n, dims), exp, err_msg=sc)
    g = q.lfsr_generator_vector(0xACE1, max(dims, 2))[:dims]
    sh = [0x12345 * (j + 3) & 0xFFFFFFFF for j in range(dims)]
    got = u32(q.lattice_fill(n, g, first=first, shifts=sh, fixed=True)).reshape(n, dims)
    i = (np.arange(first, first + n, dtype=np.uint64) & 0xFFFFFFFF).astype(np.uint32)
    br = np.array([int("{:032b}".format(int(v))[::-1], 2) for v in i], np.uint64)
    exp = ((br[:, None] * np.array(g, np.uint64)[None, :] + np.array(sh, np.uint64)[None, :])
           & 0xFFFFFFFF).astype(np.uint32)
    np.testing.assert_array_equal(got, exp)
