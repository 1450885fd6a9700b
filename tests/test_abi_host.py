"""CPU-side checks of the product library: it loads without a GPU, exports
every symbol include/qmcgpu.h declares, and its host-setup functions (tables
the reference also builds on the host) match the oracle / reference. No
per-sample compute is called here."""
import os
import re

import numpy as np
import pytest

import paper_2307_15584_b200 as q
from oracle import ptr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "qmcgpu.h")).read()
    names = sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(qmc_[a-z0-9_]+)\(", hdr, re.M)))
    assert len(names) >= 29
    L = q.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.qmc_abi_version() == 1


def test_library_exports_only_the_c_abi():
    """exports.map: the dynamic symbol table is exactly the header's qmc_*
    functions (no C++ internals, no static cudart)."""
    import shutil
    import subprocess

    if shutil.which("nm") is None:
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--defined-only", q.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    hdr = open(os.path.join(ROOT, "include", "qmcgpu.h")).read()
    names = set(re.findall(r"^[A-Za-z_][\w \*]*?\b(qmc_[a-z0-9_]+)\(", hdr, re.M))
    assert sorted(s for s in syms if s not in names) == []


def test_primes_and_max_powers(golden_arrays):
    for k in [0, 1, 2, 10, 500, 999]:
        assert q.prime(k) == golden_arrays["primes"][k]
        assert q.prime_max_power(k) == golden_arrays["prime_max_powers"][k]
    with pytest.raises(IndexError):
        q.prime(1000)
    assert q.prime_max_power(0) == 1 << 31 and q.prime_max_power(1) == 3486784401


def test_faure_and_factors(golden):
    for b in range(2, 32):
        assert q.faure_permutation(b) == golden["faure"][str(b)]
    with pytest.raises(ValueError):
        q.faure_permutation(1)
    assert q.default_linear_factors(5) == [1, 2, 4, 6, 10]


def test_lfsr_pixel_hash(golden_arrays, golden):
    assert q.lfsr_generator_vector(0xACE1, 16) == golden_arrays["lfsr_ace1_16"].tolist()
    with pytest.raises(ValueError):
        q.lfsr_generator_vector(0, 4)
    for j, x, y, h in golden["pixel_hash_probes"]:
        assert q.pixel_hash(j, x, y) == h


def test_enumeration_and_partition(golden):
    for key, rec in golden["halton_enum"].items():
        w, h = map(int, key.split("x"))
        for px, py, off in rec["offsets"]:
            e = q.halton_pixel_enumeration(w, h, px, py)
            assert e["offset"] == off and e["stride"] == rec["stride"]
            assert [e["exponent_x"], e["exponent_y"], e["scale_x"], e["scale_y"]] == rec["exps"]
    with pytest.raises(q.ConfigError):
        q.halton_pixel_enumeration((1 << 20) + 1, 2)
    for p, parts, b, rem, mod in golden["partition"]:
        assert q.partition_by_extra_dimension(p, parts, b) == (rem, mod)
    with pytest.raises(q.ConfigError):
        q.partition_by_extra_dimension(0, 6, 2)
    with pytest.raises(IndexError):
        q.partition_by_extra_dimension(4, 4, 2)
    assert q.hilbert_order_for(3840, 2160) == 12


def test_matrices(golden_arrays, golden, ref):
    m = q.GeneratorMatrixSet.builtin(64)
    np.testing.assert_array_equal(m.columns(), golden_arrays["sobol_columns64"])
    with pytest.raises(q.ConfigError):
        q.GeneratorMatrixSet.builtin(65)
    rows = golden["direction_numbers"]
    text = "d s a m_i\n" + "\n".join(
        "%d %d %d %s" % (d, s, a, " ".join(map(str, ms))) for d, s, a, ms in rows[:20]) + "\n"
    t = q.GeneratorMatrixSet.from_text(text, 21)
    np.testing.assert_array_equal(t.columns(), golden_arrays["sobol_columns64"][:21])
    # malformed files: same error class and message as the reference parser
    for bad in ["d s a\n2 1 0 2\n", "d s a\n3 1 0 1\n", "d s a\n2 1 0 1 1\n",
                "d s a\n2 2 1 1\n", "d s a\n2 2 1 1 5\n", "d s a\n2 0 0\n"]:
        with pytest.raises(q.ConfigError) as ei:
            q.GeneratorMatrixSet.from_text(bad, 2)
        cols = np.zeros((2, 52), np.uint32)
        assert ref.ref_build_matrices_text(bad.encode(), 2, ptr(cols)) == 1
        assert str(ei.value) == ref.ref_last_error().decode()


def test_sampler_names():
    for k, name in enumerate(q.SAMPLER_KINDS):
        assert q.sampler_kind_from_name(name) == k
        assert q.sampler_kind_name(k) == name
    assert q.sampler_kind_name(99) == ""
    assert q.status_string(0) == "ok" and q.status_string(1) == "config error"
    with pytest.raises(q.ConfigError):
        q.sampler_kind_from_name("sobol2")


def test_div32_magic_host_emulation():
    """The device's exact division (device.cuh div32 / internal.hpp
    make_div32), emulated in numpy for every divisor the kernels use."""
    def make(d):
        l = 0
        while (1 << l) < d:
            l += 1
        return ((1 << 32) * ((1 << l) - d)) // d + 1, l - 1

    rng = np.random.default_rng(0)
    n = np.concatenate([rng.integers(0, 1 << 32, 20000, dtype=np.uint64),
                        np.array([0, 1, 2, 3, (1 << 32) - 1, (1 << 32) - 2, 1 << 31], np.uint64)])
    ds = [q.prime(k) for k in range(0, 1000, 7)] + [q.prime_max_power(k) for k in range(0, 1000, 7)]
    ds += [2, 3, 4, 5, 7, 32, 48, 100, 128, 1000, (1 << 31) + 1, (1 << 32) - 1]
    for d in ds:
        m, s = make(d)
        t = (n * np.uint64(m)) >> np.uint64(32)
        qq = (t + ((n - t) >> np.uint64(1))) >> np.uint64(s)
        np.testing.assert_array_equal(qq, n // np.uint64(d))


def test_frac_div_magic_host_emulation():
    """device.cuh frac_div_magic: floor(acc * 2^32 / scale) from
    m = floor(2^64 / scale) (pow_magic) with one 64-bit check, emulated with
    Python integers for every divisor family the kernels use: b^D for the
    first 1000 primes (all D with b^D < 2^32), acc at the edges and random."""
    rng = np.random.default_rng(1)
    scales = set()
    for k in range(0, 1000, 3):
        b, p = q.prime(k), q.prime(k)
        while p < (1 << 32):
            scales.add(p)
            p *= b
    scales.discard(2)
    scales = sorted(s for s in scales if s & 1)  # base 2 never divides (brev path)
    checked = 0
    for s in scales:
        m = ((1 << 64) - 1) // s
        mlo, mhi = m & 0xFFFFFFFF, m >> 32
        accs = {0, 1, s - 1, s // 2, (s - 1) // 3} | {int(a) for a in rng.integers(0, s, 12)}
        for acc in accs:
            qe = (acc * mhi + ((acc * mlo) >> 32)) & 0xFFFFFFFF
            if (qe + 1) * s <= acc << 32:
                qe += 1
            assert qe == (acc << 32) // s, (acc, s)
            checked += 1
    assert checked > 5000


GV_CASES = ["1\n3\n5\n", "# header\n1 # first\n\n1276675999\n", "7", "1\n4\n", "1\n4294967297\n",
            "# only comments\n\n", "1\n  3  \n"]
FACTOR_CASES = ["3 2\n5 3\n", "# c\n7 6\n\n", "2 1\n", "3\n", "3 0\n", "3 3\n", "1 0\n",
                "997 5\n"]


@pytest.mark.parametrize("text", GV_CASES)
def test_load_generator_vector_matches_reference(ref, text):
    import ctypes as C
    n = C.c_uint32()
    out = np.zeros(16, np.uint32)
    rc = ref.ref_load_generator_vector(text.encode(), ptr(out), 16, C.byref(n))
    if rc != 0:
        with pytest.raises(q.ConfigError) as ei:
            q.load_generator_vector(text)
        assert str(ei.value) == ref.ref_last_error().decode()
    else:
        assert q.load_generator_vector(text) == out[: n.value].tolist()


@pytest.mark.parametrize("text", FACTOR_CASES)
def test_load_linear_factors_matches_reference(ref, text):
    out = np.zeros(200, np.uint32)
    rc = ref.ref_load_linear_factors(text.encode(), 200, ptr(out))
    if rc != 0:
        with pytest.raises(q.ConfigError) as ei:
            q.load_linear_factors(text, 200)
        assert str(ei.value) == ref.ref_last_error().decode()
    else:
        assert q.load_linear_factors(text, 200) == out.tolist()


def test_fnv1a64(golden):
    assert q.fnv1a64(b"") == 0xCBF29CE484222325
    assert q.fnv1a64(b"a") == 0xAF63DC4C8601EC8C


def test_points_csv_format_host():
    """sobol N=4 dims=2 CSV -> 4 lines, first "0.000000000,0.000000000"."""
    pts = np.array([[0.0, 0.0], [0.5, 0.5], [0.75, 0.25], [0.25, 0.75]], np.float32)
    text = q.write_points_csv(pts).decode()
    lines = text.splitlines()
    assert len(lines) == 4 and lines[0] == "0.000000000,0.000000000"
    assert lines[2] == "0.750000000,0.250000000"
    rng = np.random.default_rng(0)
    x = rng.random((50, 3)).astype(np.float32)
    assert q.write_points_csv(x).decode() == "".join(
        ",".join("%.9f" % v for v in row) + "\n" for row in x.astype(np.float64))


def test_hilbert_digit_reverse_lattice_shift_vs_reference(ref):
    """Host helpers of the lattice / image-plane family against the
    reference: values and exception classes (status codes match the shim's)."""
    import ctypes as C

    rng = np.random.default_rng(11)
    L = q.lib()
    for order in (1, 2, 5, 12, 16, 31):
        n = 1 << order
        for x, y in [(0, 0), (n - 1, n - 1)] + [tuple(int(v) for v in rng.integers(0, n, 2))
                                                for _ in range(50)]:
            d, e = C.c_uint64(), C.c_uint64()
            assert ref.ref_hilbert_index(x, y, order, C.byref(e)) == 0
            assert q.hilbert_index(x, y, order) == e.value
            assert q.hilbert_xy(e.value, order) == (x, y)
        for dd in [0, (1 << (2 * order)) - 1] + [int(v) for v in rng.integers(0, 1 << (2 * order),
                                                                               20, dtype=np.uint64)]:
            rx, ry = C.c_uint32(), C.c_uint32()
            assert ref.ref_hilbert_xy(dd, order, C.byref(rx), C.byref(ry)) == 0
            assert q.hilbert_xy(dd, order) == (rx.value, ry.value)
    for args in [(0, 0, 0), (0, 0, 32), (2, 0, 1), (0, 4, 2)]:
        d, e = C.c_uint64(), C.c_uint64()
        assert L.qmc_hilbert_index(*args, C.byref(d)) == ref.ref_hilbert_index(*args, C.byref(e))
    for args in [(0, 0), (4, 1), (16, 2)]:
        a, b = C.c_uint32(), C.c_uint32()
        assert L.qmc_hilbert_xy(*args, C.byref(a), C.byref(b)) == \
            ref.ref_hilbert_xy(*args, C.byref(a), C.byref(b))
    for v, b, k in [(0, 2, 0), (5, 2, 3), (12345678901, 3, 22), (2**64 - 1, 7, 20), (99, 10, 2)]:
        assert q.digit_reverse(v, b, k) == ref.ref_digit_reverse(v, b, k)
    g = np.array(q.lfsr_generator_vector(0xACE1, 8), np.uint32)
    for k, m in [(0, 0), (1, 1), (3, 10), (5, 29), (1, 31), (0, 32)]:
        exp = np.zeros(8, np.uint32)
        assert ref.ref_lattice_shift_fixed(k, m, g.ctypes.data, 8, exp.ctypes.data) == 0
        assert q.lattice_shift_fixed(k, m, g) == exp.tolist()
    out = np.zeros(8, np.uint32)
    for k, m in [(1, 33), (1, 32), (2, 32), (1 << 20, 20)]:
        assert L.qmc_lattice_shift_fixed(k, m, g.ctypes.data, 8, out.ctypes.data) == \
            ref.ref_lattice_shift_fixed(k, m, g.ctypes.data, 8, out.ctypes.data) != 0


def test_reduce_deterministic_vs_reference(ref):
    """reduce_deterministic (quality.cpp:158-166): rank-sorted CompensatedSum,
    bit-identical for shuffled ranks and values spanning many magnitudes."""
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 1000, 20000):
        ranks = rng.permutation(n).astype(np.uint32)
        vals = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n)
        got = q.reduce_deterministic(ranks, vals)
        exp = ref.ref_reduce_deterministic(ranks.ctypes.data, vals.ctypes.data, n)
        assert got == exp or (np.isnan(got) and np.isnan(exp)), n


def test_hilbert_state_tables_match_generator():
    """device.cuh's kHilbert3 / kHilbert1 are the state machine that
    tools/gen_hilbert_table.py derives from hilbert.hpp's per-level rule (and
    checks against it); the library's hilbert_index is compared with the
    reference in test_hilbert_digit_reverse_lattice_shift_vs_reference."""
    import importlib.util
    import re

    spec = importlib.util.spec_from_file_location(
        "gen_hilbert_table", os.path.join(ROOT, "tools", "gen_hilbert_table.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    t3, t1 = g.tables()
    src = open(os.path.join(ROOT, "paper_2307_15584_b200", "csrc", "device.cuh")).read()
    block = src[src.index("#define QMC_HILBERT3"):src.index("#define QMC_HILBERT1")]
    assert [int(v) for v in re.findall(r"\b\d+\b", block.split("{", 1)[1])] == t3
    m = re.search(r"#define QMC_HILBERT1 \{([^}]*)\}", src)
    assert [int(v) for v in m.group(1).split(",")] == t1
    rng = np.random.default_rng(3)
    for order in (1, 3, 4, 7, 12, 13, 31):
        n = 1 << order
        for x, y in rng.integers(0, n, (200, 2), dtype=np.uint64):
            assert g.fast_index(int(x), int(y), order, t3, t1) == g.ref_index(int(x), int(y), order)


def test_hilbert_phi3_fixed_vs_reference(ref, golden):
    """hilbert_phi3_fixed (imageplane.cpp:16-21) at random pixels of every
    order, including indices past 3^20 (the table's index modulus)."""
    import ctypes as C

    rng = np.random.default_rng(9)
    for order in (1, 2, 5, 12, 16, 17, 24, 31):
        n = 1 << order
        for x, y in rng.integers(0, n, (100, 2), dtype=np.uint64):
            e = C.c_uint32()
            assert ref.ref_hilbert_phi3_fixed(int(x), int(y), order, C.byref(e)) == 0
            assert q.hilbert_phi3_fixed(int(x), int(y), order) == e.value
    with pytest.raises(ValueError):
        q.hilbert_phi3_fixed(0, 0, 0)
    with pytest.raises(IndexError):
        q.hilbert_phi3_fixed(4, 0, 2)


def test_nccl_loads_lazily_without_a_gpu():
    """The library binds NCCL on first use (no link-time dependency): the
    version query works here; communicator calls fail with a status, not a
    crash, when no GPU is present."""
    v = q.nccl_version()
    assert v >= 22700, v
    with pytest.raises((q.CudaError, RuntimeError)):
        q.Comm.init_all([0])
    with pytest.raises(ValueError):
        q.Comm.init_rank(b"x" * 7, 1, 0)


def test_render_output_validation():
    """Caller-supplied render outputs are checked before the C-ABI writes
    rows * width elements (dtype, size, contiguity)."""
    with pytest.raises(ValueError):
        q.render_devices(8, 4, 1, [0], out=np.empty((3, 8), np.float32))
    with pytest.raises(ValueError):
        q.render_devices(8, 4, 1, [0], out=np.empty((4, 8), np.float64))
    with pytest.raises(ValueError):
        q.render_samples_devices(8, 4, 1, [0], out=np.empty((8, 8), np.float32)[:, ::2])
    with pytest.raises(ValueError):
        q.render_nccl_devices(8, 4, 1, [0], out=np.empty(31, np.float32))
