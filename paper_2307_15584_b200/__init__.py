"""B200-native QMC sampling path (arXiv 2307.15584) — Python host binding.

Thin ctypes layer over ``libqmcgpu.so`` (the C-ABI in ``include/qmcgpu.h``;
sm_100a kernels in ``csrc/``). Names mirror the reference library's ``qmc::``
surface (/root/reference/proj/include/qmc/*.hpp) so tests read like the
reference's own obligations; errors map to the reference's exception classes:

    qmc::ConfigError        -> ConfigError (RuntimeError)
    std::invalid_argument   -> ValueError
    std::out_of_range       -> IndexError
    std::overflow_error     -> OverflowError
    CUDA failure / no GPU   -> CudaError (RuntimeError)

There is no CPU fallback: every per-sample computation runs in the CUDA
library, and importing this package fails loudly when the library is missing.
Device outputs are torch tensors on the current CUDA device; host (numpy)
outputs go through the library's chunked D2H pipeline.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqmcgpu.so")

__all__ = [
    "ConfigError", "CudaError", "lib", "GeneratorMatrixSet", "map_u32_to_unifloat",
    "map_selfcheck", "sobol_fill", "halton_fill", "radical_inverse_fill", "lattice_fill",
    "stream_fill", "render", "scene_value", "prime", "prime_max_power", "faure_permutation",
    "default_linear_factors", "lfsr_generator_vector", "pixel_hash", "hilbert_order_for",
    "partition_by_extra_dimension", "halton_pixel_enumeration", "sampler_kind_from_name",
    "integrate", "builtin_integrand", "write_probe", "l2_star_discrepancy",
    "min_toroidal_distance", "check_1d_stratification", "XorTables", "render_partial",
    "render_finalize", "load_generator_vector", "load_linear_factors", "fnv1a64", "write_pnm",
    "write_points_csv", "hilbert_index", "hilbert_xy", "hilbert_phi3_fixed", "digit_reverse", "lattice_shift_fixed",
    "integrate_partials", "reduce_deterministic", "render_devices", "render_samples_devices", "sampler_kind_name", "status_string",
    "SAMPLER_KINDS", "run_bench_kernel", "fp64_probe", "Comm", "nccl_version", "render_nccl", "render_nccl_devices",
]


class ConfigError(RuntimeError):
    """qmc::ConfigError (errors.hpp:13-15)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside libqmcgpu."""


SAMPLER_KINDS = ["sobol", "halton", "lattice", "halton-hilbert", "pixel-shifted-lattice",
                 "pixel-random-lattice", "image-plane-halton", "sobol-xor-table"]

u32, u64, i32, f64, P = C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_void_p


class StreamParams(C.Structure):
    _fields_ = [("dims", u32), ("generator", P), ("generator_dims", u32), ("matrices", P),
                ("sobol_scrambles", P), ("sobol_scrambles_len", u32), ("halton_scramble", u32),
                ("linear_factors", P), ("linear_factors_len", u32), ("px", u32), ("py", u32),
                ("order", u32), ("spp", u32), ("width", u32), ("height", u32),
                ("xor_seed", u32), ("xor_point_count", u32), ("xor_tables", P)]


class RenderJob(C.Structure):
    _fields_ = [("width", u32), ("height", u32), ("spp", u32), ("kind", i32), ("accum", i32),
                ("seed", u32), ("generator", P), ("generator_dims", u32), ("matrices", P),
                ("tables", P)]


class IntegrationRow(C.Structure):
    _fields_ = [("n", u64), ("estimate", f64), ("abs_error", f64), ("seconds", f64)]


class BenchResult(C.Structure):
    _fields_ = [("evaluations", u64), ("seconds", f64), ("components_per_second", f64),
                ("checksum", u64)]


class HaltonEnumeration(C.Structure):
    _fields_ = [("scale_x", u32), ("scale_y", u32), ("exponent_x", u32), ("exponent_y", u32),
                ("stride", u64)]


_lib = None


def lib():
    """Load libqmcgpu.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            "libqmcgpu.so not built (%s); run `python -c 'import __graft_entry__ as g; g.build()'`"
            % LIB_PATH)
    L = C.CDLL(LIB_PATH)

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype, f.argtypes = res, list(args)

    sig("qmc_last_error", C.c_char_p)
    sig("qmc_status_string", C.c_char_p, i32)
    sig("qmc_sampler_kind_name", C.c_char_p, i32)
    sig("qmc_abi_version", i32)
    sig("qmc_map_u32_to_unifloat", i32, P, P, u64, P)
    sig("qmc_map_selfcheck", i32, C.POINTER(u64), P)
    sig("qmc_write_probe", i32, P, u64, i32, P)
    sig("qmc_prime", i32, u32, C.POINTER(u32))
    sig("qmc_prime_max_power", i32, u32, C.POINTER(u32))
    sig("qmc_faure_permutation", i32, u32, P)
    sig("qmc_default_linear_factors", i32, u32, P)
    sig("qmc_lfsr_generator_vector", i32, u32, u32, P)
    sig("qmc_pixel_hash", u32, u32, u32, u32)
    sig("qmc_hilbert_order_for", u32, u32, u32)
    sig("qmc_partition_by_extra_dimension", i32, u32, u32, u32, C.POINTER(u64), C.POINTER(u64))
    sig("qmc_hilbert_index", i32, u32, u32, u32, C.POINTER(u64))
    sig("qmc_render_devices", i32, C.POINTER(RenderJob), P, u32, P)
    sig("qmc_render_samples_devices", i32, C.POINTER(RenderJob), P, u32, P)
    sig("qmc_integrate_partials", i32, i32, C.POINTER(StreamParams), i32, u32, u64, u64, u64, i32,
        P, C.POINTER(C.c_int64), P)
    sig("qmc_reduce_deterministic", i32, P, P, u64, C.POINTER(f64))
    sig("qmc_hilbert_xy", i32, u64, u32, C.POINTER(u32), C.POINTER(u32))
    sig("qmc_hilbert_phi3_fixed", i32, u32, u32, u32, C.POINTER(u32))
    sig("qmc_digit_reverse", u64, u64, u32, u32)
    sig("qmc_lattice_shift_fixed", i32, u32, u32, P, u32, P)
    sig("qmc_halton_pixel_enumeration", i32, u32, u32, u32, u32, C.POINTER(HaltonEnumeration),
        C.POINTER(u64))
    sig("qmc_matrices_builtin", i32, u32, C.POINTER(P))
    sig("qmc_matrices_from_text", i32, C.c_char_p, u32, C.POINTER(P))
    sig("qmc_matrices_from_columns", i32, P, u32, C.POINTER(P))
    sig("qmc_matrices_dims", u32, P)
    sig("qmc_matrices_columns", i32, P, P)
    sig("qmc_matrices_destroy", None, P)
    sig("qmc_sobol_fill", i32, P, u64, u64, u32, i32, P, i32, P, P)
    sig("qmc_halton_fill", i32, u64, u64, u32, i32, P, i32, P, P)
    sig("qmc_radical_inverse_fill", i32, u64, u64, u32, i32, u32, i32, P, P)
    sig("qmc_lattice_fill", i32, P, P, u32, u64, u64, i32, P, P)
    sig("qmc_sampler_kind_from_name", i32, C.c_char_p, C.POINTER(i32))
    sig("qmc_stream_fill", i32, i32, C.POINTER(StreamParams), u64, u64, i32, P, P)
    sig("qmc_render", i32, C.POINTER(RenderJob), u32, u32, P, P)
    sig("qmc_scene_value", i32, P, P, u64, P)
    sig("qmc_load_generator_vector", i32, C.c_char_p, P, u32, C.POINTER(u32))
    sig("qmc_load_linear_factors", i32, C.c_char_p, u32, P)
    sig("qmc_fnv1a64", u64, P, u64)
    sig("qmc_write_points_csv", i32, P, u64, u32, P, C.POINTER(C.c_size_t), P)
    sig("qmc_write_pnm", i32, P, u32, u32, u32, P, C.POINTER(C.c_size_t), P)
    sig("qmc_render_partial", i32, C.POINTER(RenderJob), u32, u32, u32, u32, P, P)
    sig("qmc_render_finalize", i32, P, u64, u32, P, P)
    sig("qmc_l2_star_discrepancy", i32, P, u64, u32, C.POINTER(f64), P)
    sig("qmc_min_toroidal_distance", i32, P, u64, u32, C.POINTER(f64), P)
    sig("qmc_check_1d_stratification", i32, i32, C.POINTER(StreamParams), u32, u32,
        C.POINTER(i32), P, P)
    sig("qmc_xor_tables_white_noise", i32, u32, u32, u32, C.POINTER(P))
    sig("qmc_xor_tables_load", i32, P, C.c_size_t, u32, P, u32, C.POINTER(P))
    sig("qmc_xor_tables_write", i32, P, P, C.POINTER(C.c_size_t))
    sig("qmc_xor_tables_dims", u32, P)
    sig("qmc_xor_tables_point_count", u32, P)
    sig("qmc_xor_tables_destroy", None, P)
    sig("qmc_builtin_integrand", i32, C.c_char_p, u32, C.POINTER(i32), C.POINTER(f64))
    sig("qmc_integrate", i32, i32, C.POINTER(StreamParams), i32, u32, u64, i32,
        C.POINTER(IntegrationRow), P)
    sig("qmc_run_bench_kernel", i32, C.c_char_p, u64, u32, C.POINTER(BenchResult), P)
    sig("qmc_fp64_probe", i32, u32, C.POINTER(f64), P)
    sig("qmc_nccl_version", i32, C.POINTER(i32))
    sig("qmc_comm_unique_id", i32, P)
    sig("qmc_comm_init_rank", i32, P, i32, i32, C.POINTER(P))
    sig("qmc_comm_init_all", i32, P, i32, P)
    sig("qmc_comm_from_nccl", i32, P, C.POINTER(P))
    sig("qmc_comm_info", i32, P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32))
    sig("qmc_comm_destroy", None, P)
    sig("qmc_render_nccl", i32, C.POINTER(RenderJob), P, i32, P, P)
    sig("qmc_render_nccl_devices", i32, C.POINTER(RenderJob), P, u32, i32, P)
    _lib = L
    return L


_ERRORS = {1: ConfigError, 2: ValueError, 3: IndexError, 4: OverflowError, 5: CudaError,
           6: CudaError, 9: RuntimeError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().qmc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ----------------------------------------------------------------- helpers
def _torch():
    import torch

    return torch


def _stream(stream) -> Optional[int]:
    if stream is not None:
        return int(stream)
    torch = _torch()
    if torch.cuda.is_available():
        return torch.cuda.current_stream().cuda_stream
    return None


def _u32_host(a, n=None) -> Optional[np.ndarray]:
    if a is None:
        return None
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint64) & 0xFFFFFFFF, dtype=np.uint32)
    if n is not None and arr.size < n:
        raise ValueError("array shorter than dims")
    return arr


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _alloc(n: int, dims: int, fixed: bool, out, device=None):
    """Output buffer: given (torch tensor / numpy array) or a new CUDA tensor."""
    if out is not None:
        nbytes = out.nbytes if isinstance(out, np.ndarray) else out.numel() * out.element_size()
        if nbytes < n * dims * 4:
            raise ValueError("output buffer too small")
        return out
    torch = _torch()
    dt = torch.int32 if fixed else torch.float32
    shape = (n, dims) if dims != 1 else (n,)
    return torch.empty(shape, dtype=dt, device=device or "cuda")


def _check_out(out, count: int, dtype: str):
    """A caller-supplied render output must hold `count` C-contiguous elements
    of `dtype` ("float32" / "int64"): the C-ABI writes exactly that many."""
    if isinstance(out, np.ndarray):
        ok_dt = out.dtype == np.dtype(dtype)
        contig = out.flags["C_CONTIGUOUS"]
        nbytes = out.nbytes
        size = out.size
    else:
        ok_dt = str(out.dtype) == "torch." + dtype
        contig = out.is_contiguous()
        size = out.numel()
        nbytes = size * out.element_size()
    if not ok_dt:
        raise ValueError("output must be %s, got %s" % (dtype, out.dtype))
    if not contig:
        raise ValueError("output must be C-contiguous")
    if size < count or nbytes < count * np.dtype(dtype).itemsize:
        raise ValueError("output buffer too small: %d elements for %d" % (size, count))
    return out


_SOBOL = {"none": 0, "plain": 0, "xor": 1, "owen": 2}
_RADICAL = {"plain": 0, "linear": 1, "faure": 2}
_ACCUM = {"kahan": 0, "int": 1}


# ---------------------------------------------------------------- host setup
def prime(index: int) -> int:
    o = u32()
    _check(lib().qmc_prime(index, C.byref(o)))
    return o.value


def prime_max_power(index: int) -> int:
    o = u32()
    _check(lib().qmc_prime_max_power(index, C.byref(o)))
    return o.value


def faure_permutation(base: int) -> list:
    out = np.zeros(max(base, 1), np.uint32)
    _check(lib().qmc_faure_permutation(base, out.ctypes.data))
    return out.tolist()


def default_linear_factors(dims: int) -> list:
    out = np.zeros(max(dims, 1), np.uint32)
    _check(lib().qmc_default_linear_factors(dims, out.ctypes.data))
    return out[:dims].tolist()


def lfsr_generator_vector(seed: int, dims: int) -> list:
    out = np.zeros(max(dims, 1), np.uint32)
    _check(lib().qmc_lfsr_generator_vector(seed, dims, out.ctypes.data))
    return out[:dims].tolist()


def pixel_hash(j: int, px: int, py: int) -> int:
    return lib().qmc_pixel_hash(j, px, py)


def hilbert_order_for(width: int, height: int) -> int:
    return lib().qmc_hilbert_order_for(width, height)


def partition_by_extra_dimension(part: int, parts: int, base: int):
    r, m = u64(), u64()
    _check(lib().qmc_partition_by_extra_dimension(part, parts, base, C.byref(r), C.byref(m)))
    return r.value, m.value


def hilbert_index(x: int, y: int, order: int) -> int:
    """hilbert_index(PixelCoord{x, y, order}) (hilbert.hpp:39-56)."""
    d = u64()
    _check(lib().qmc_hilbert_index(x, y, order, C.byref(d)))
    return d.value


def hilbert_phi3_fixed(x: int, y: int, order: int) -> int:
    """hilbert_phi3_fixed(PixelCoord{x, y, order}) (imageplane.cpp:16-21)."""
    o = u32()
    _check(lib().qmc_hilbert_phi3_fixed(x, y, order, C.byref(o)))
    return o.value


def hilbert_xy(d: int, order: int):
    """hilbert_xy(d, order) -> (x, y) (hilbert.hpp:59-78)."""
    x, y = u32(), u32()
    _check(lib().qmc_hilbert_xy(d, order, C.byref(x), C.byref(y)))
    return x.value, y.value


def digit_reverse(v: int, base: int, digits: int) -> int:
    """digit_reverse (imageplane.cpp:43-51)."""
    return lib().qmc_digit_reverse(v, base, digits)


def lattice_shift_fixed(k: int, m: int, g) -> list:
    """lattice_shift_fixed(k, m, g) (lattice.cpp:157-170): the integer shift
    mapping block 0 of 2^m points onto block k (qmc_lattice_fill `shifts`)."""
    gv = _u32_host(g)
    out = np.zeros(max(gv.size, 1), np.uint32)
    _check(lib().qmc_lattice_shift_fixed(k, m, gv.ctypes.data, gv.size, out.ctypes.data))
    return out[:gv.size].tolist()


def halton_pixel_enumeration(width: int, height: int, px: int = 0, py: int = 0):
    e, off = HaltonEnumeration(), u64()
    _check(lib().qmc_halton_pixel_enumeration(width, height, px, py, C.byref(e), C.byref(off)))
    return {"scale_x": e.scale_x, "scale_y": e.scale_y, "exponent_x": e.exponent_x,
            "exponent_y": e.exponent_y, "stride": e.stride, "offset": off.value}


def sampler_kind_from_name(name: str) -> int:
    o = i32()
    _check(lib().qmc_sampler_kind_from_name(name.encode(), C.byref(o)))
    return o.value


def sampler_kind_name(kind: int) -> str:
    """sampler_kind_name (imageplane.cpp:273-284); "" for an unknown value."""
    return lib().qmc_sampler_kind_name(kind).decode()


def status_string(status: int) -> str:
    """Human-readable name of a qmc_status code."""
    return lib().qmc_status_string(status).decode()


class GeneratorMatrixSet:
    """Immutable Sobol' generator matrices (digitalnet.hpp:50-63) in libqmcgpu."""

    def __init__(self, handle: int):
        self._h = handle

    @classmethod
    def builtin(cls, dims: int) -> "GeneratorMatrixSet":
        h = P()
        _check(lib().qmc_matrices_builtin(dims, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_text(cls, text: str, dims: int) -> "GeneratorMatrixSet":
        h = P()
        _check(lib().qmc_matrices_from_text(text.encode(), dims, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_columns(cls, columns) -> "GeneratorMatrixSet":
        c = np.ascontiguousarray(columns, dtype=np.uint32)
        h = P()
        _check(lib().qmc_matrices_from_columns(c.ctypes.data, c.shape[0], C.byref(h)))
        return cls(h.value)

    @property
    def dims(self) -> int:
        return lib().qmc_matrices_dims(self._h)

    def columns(self) -> np.ndarray:
        out = np.zeros((self.dims, 52), np.uint32)
        _check(lib().qmc_matrices_columns(self._h, out.ctypes.data))
        return out

    @property
    def handle(self) -> int:
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.qmc_matrices_destroy(self._h)
            self._h = None


class XorTables:
    """XOR-table sampler data (imageplane.hpp:92-120) held by libqmcgpu."""

    def __init__(self, handle: int):
        self._h = handle

    @classmethod
    def white_noise(cls, dims: int, point_count: int, seed: int) -> "XorTables":
        """white_noise_xor_tables (imageplane.cpp:197-229)."""
        h = P()
        _check(lib().qmc_xor_tables_white_noise(dims, point_count, seed, C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, data: bytes, dims: int, points, point_count: int) -> "XorTables":
        """load_xor_tables from an XQT1 file image (imageplane.cpp:163-195)."""
        pts = _u32_host(points)
        if pts.size != point_count * dims:
            raise ConfigError("load_xor_tables: point set size does not match point_count * dims")
        buf = C.create_string_buffer(bytes(data), len(data))
        h = P()
        _check(lib().qmc_xor_tables_load(buf, len(data), dims, pts.ctypes.data, point_count,
                                         C.byref(h)))
        return cls(h.value)

    def to_bytes(self) -> bytes:
        """write_xor_table_file (imageplane.cpp:154-161)."""
        n = C.c_size_t(0)
        _check(lib().qmc_xor_tables_write(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib().qmc_xor_tables_write(self._h, buf, C.byref(n)))
        return buf.raw[: n.value]

    @property
    def dims(self) -> int:
        return lib().qmc_xor_tables_dims(self._h)

    @property
    def point_count(self) -> int:
        return lib().qmc_xor_tables_point_count(self._h)

    @property
    def handle(self) -> int:
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.qmc_xor_tables_destroy(self._h)
            self._h = None


_builtin_cache: dict = {}


def _builtin(dims: int) -> GeneratorMatrixSet:
    m = _builtin_cache.get(dims)
    if m is None:
        m = _builtin_cache[dims] = GeneratorMatrixSet.builtin(dims)
    return m


# ------------------------------------------------------------------ fills
def map_u32_to_unifloat(x, out=None, stream=None):
    """Bit-exact map_u32_to_unifloat (unitfloat.hpp:34-50) over a u32 array."""
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.uint32)
        out = np.empty(x.shape, np.float32) if out is None else out
    else:
        torch = _torch()
        out = torch.empty(x.shape, dtype=torch.float32, device=x.device) if out is None else out
    _check(lib().qmc_map_u32_to_unifloat(_ptr(x), _ptr(out), int(np.prod(x.shape)), _stream(stream)))
    return out


def map_selfcheck(stream=None) -> int:
    """Exhaustive 2^32 comparison of the device map with the reference formula."""
    m = u64()
    _check(lib().qmc_map_selfcheck(C.byref(m), _stream(stream)))
    return m.value


def write_probe(buf, mode: int = 0, stream=None) -> None:
    """Write-only store stream over a device tensor (roofline diagnostic)."""
    _check(lib().qmc_write_probe(_ptr(buf), buf.numel() * buf.element_size(), mode,
                                 _stream(stream)))


def sobol_fill(n: int, dims: int, first: int = 0, scramble: str = "none", words=None,
               matrices: Optional[GeneratorMatrixSet] = None, fixed: bool = False, out=None,
               stream=None):
    """Sobol' points [n][dims] (digitalnet.cpp:111-151); scramble none|xor|owen."""
    m = matrices or _builtin(dims)
    w = _u32_host(words, dims)
    o = _alloc(n, dims, fixed, out)
    _check(lib().qmc_sobol_fill(m.handle, first, n, dims, _SOBOL[scramble], _ptr(w),
                                1 if fixed else 0, _ptr(o), _stream(stream)))
    return o


def halton_fill(n: int, dims: int, first: int = 0, scramble: str = "plain", factors=None,
                fixed: bool = False, out=None, stream=None):
    """Halton points (radical.cpp:240-269) with plain/linear/faure digit scrambles."""
    f = _u32_host(factors, dims)
    o = _alloc(n, dims, fixed, out)
    _check(lib().qmc_halton_fill(first, n, dims, _RADICAL[scramble], _ptr(f),
                                 1 if fixed else 0, _ptr(o), _stream(stream)))
    return o


def radical_inverse_fill(n: int, prime_index: int = 0, first: int = 0, scramble: str = "plain",
                         factor: int = 1, fixed: bool = False, out=None, stream=None):
    """radical_inverse*(i, prime_index) for i in [first, first+n) (radical.cpp:130-213)."""
    o = _alloc(n, 1, fixed, out)
    _check(lib().qmc_radical_inverse_fill(first, n, prime_index, _RADICAL[scramble], factor,
                                          1 if fixed else 0, _ptr(o), _stream(stream)))
    return o


def lattice_fill(n: int, g: Sequence[int], first: int = 0, shifts=None, dims: Optional[int] = None,
                 fixed: bool = False, out=None, stream=None):
    """Rank-1 lattice brev(i)*g_j (+ integer CP shift s_j) (lattice.hpp:31-39)."""
    dims = len(g) if dims is None else dims
    gv = _u32_host(g, dims)
    sv = _u32_host(shifts, dims)
    o = _alloc(n, dims, fixed, out)
    _check(lib().qmc_lattice_fill(_ptr(gv), _ptr(sv), dims, first, n, 1 if fixed else 0,
                                  _ptr(o), _stream(stream)))
    return o


def stream_fill(kind: str, n: int, dims: int = 2, first: int = 0, *, generator=None,
                matrices: Optional[GeneratorMatrixSet] = None, sobol_scrambles=None,
                scramble: str = "plain", linear_factors=None, pixel=(0, 0), order: int = 1,
                spp: int = 1, width: int = 0, height: int = 0, xor_seed: int = 0,
                xor_point_count: int = 1, xor_tables: Optional["XorTables"] = None,
                fixed: bool = False, out=None, stream=None):
    """make_stream(kind, params) + SampleStream::sample(i, j) (imageplane.cpp:310-461)."""
    k = sampler_kind_from_name(kind)
    p, keep = _stream_params(dims, generator, matrices, sobol_scrambles, scramble, linear_factors,
                             pixel, order, spp, width, height, xor_seed, xor_point_count,
                             xor_tables)
    o = _alloc(n, dims, fixed, out)
    _check(lib().qmc_stream_fill(k, C.byref(p), first, n, 1 if fixed else 0, _ptr(o),
                                 _stream(stream)))
    return o


def _stream_params(dims, generator, matrices, sobol_scrambles, scramble, linear_factors, pixel,
                   order, spp, width, height, xor_seed, xor_point_count, xor_tables=None):
    if scramble not in _RADICAL:
        raise ConfigError("make_stream: scramble must be plain, faure, or linear")
    keep = []
    p = StreamParams()
    p.dims = dims
    if generator is not None:
        g = _u32_host(generator)
        keep.append(g)
        p.generator, p.generator_dims = g.ctypes.data, g.size
    if matrices is not None:
        p.matrices = matrices.handle
    if sobol_scrambles is not None:
        s = _u32_host(sobol_scrambles)
        keep.append(s)
        p.sobol_scrambles, p.sobol_scrambles_len = s.ctypes.data, s.size
    p.halton_scramble = _RADICAL[scramble]
    if linear_factors is not None:
        f = _u32_host(linear_factors)
        keep.append(f)
        p.linear_factors, p.linear_factors_len = f.ctypes.data, f.size
    p.px, p.py = pixel
    p.order, p.spp, p.width, p.height = order, spp, width, height
    p.xor_seed, p.xor_point_count = xor_seed, xor_point_count
    if xor_tables is not None:
        p.xor_tables = xor_tables.handle
        keep.append(xor_tables)
    return p, keep


def l2_star_discrepancy(points, stream=None) -> float:
    """Warnock L2-star discrepancy of an [n, dims] float32 point set (quality.cpp:76-114)."""
    pts = np.ascontiguousarray(points, dtype=np.float32) if isinstance(points, np.ndarray) \
        else points.contiguous()
    out = f64()
    _check(lib().qmc_l2_star_discrepancy(_ptr(pts), pts.shape[0], pts.shape[1], C.byref(out),
                                         _stream(stream)))
    return out.value


def min_toroidal_distance(points, stream=None) -> float:
    """Minimum pairwise wrap-around distance (quality.cpp:116-136)."""
    pts = np.ascontiguousarray(points, dtype=np.float32) if isinstance(points, np.ndarray) \
        else points.contiguous()
    out = f64()
    _check(lib().qmc_min_toroidal_distance(_ptr(pts), pts.shape[0], pts.shape[1], C.byref(out),
                                           _stream(stream)))
    return out.value


def check_1d_stratification(kind: str, j: int, m: int, dims: int = 2, *, generator=None,
                            matrices: Optional[GeneratorMatrixSet] = None, sobol_scrambles=None,
                            scramble: str = "plain", linear_factors=None, pixel=(0, 0),
                            order: int = 1, spp: int = 1, width: int = 0, height: int = 0,
                            xor_seed: int = 0, xor_point_count: int = 1, stream=None):
    """(ok, histogram) of check_1d_stratification(make_stream(kind, ...), j, m)."""
    k = sampler_kind_from_name(kind)
    p, keep = _stream_params(dims, generator, matrices, sobol_scrambles, scramble, linear_factors,
                             pixel, order, spp, width, height, xor_seed, xor_point_count)
    ok = i32()
    hist = np.zeros(1 << min(m, 20), np.uint32)
    _check(lib().qmc_check_1d_stratification(k, C.byref(p), j, m, C.byref(ok), hist.ctypes.data,
                                             _stream(stream)))
    return bool(ok.value), hist


_INTEGRANDS = {"product-sine": 0, "product-poly": 1, "indicator": 2}


def builtin_integrand(name: str, dims: int):
    """(id, exact integral) of builtin_integrand(name, dims) (quality.cpp:28-74)."""
    k, ex = i32(), f64()
    _check(lib().qmc_builtin_integrand(name.encode(), dims, C.byref(k), C.byref(ex)))
    return k.value, ex.value


def integrate(kind: str, integrand: str, n: int, dims: int, accum: str = "kahan", *,
              stream_dims: Optional[int] = None, generator=None,
              matrices: Optional[GeneratorMatrixSet] = None, sobol_scrambles=None,
              scramble: str = "plain", linear_factors=None, pixel=(0, 0), order: int = 1,
              spp: int = 1, width: int = 0, height: int = 0, xor_seed: int = 0,
              xor_point_count: int = 1, stream=None) -> dict:
    """integrate(make_stream(kind, ...), builtin_integrand(integrand, dims), n, accum)
    (quality.cpp:214-282); returns the IntegrationRow fields as a dict."""
    k = sampler_kind_from_name(kind)
    if accum not in _ACCUM:
        raise ConfigError("accumulation mode must be 'kahan' or 'int'")
    if integrand not in _INTEGRANDS:
        raise ConfigError("unknown integrand: " + integrand)
    sd = dims if stream_dims is None else stream_dims
    p, keep = _stream_params(sd, generator, matrices, sobol_scrambles, scramble, linear_factors,
                             pixel, order, spp, width, height, xor_seed, xor_point_count)
    row = IntegrationRow()
    _check(lib().qmc_integrate(k, C.byref(p), _INTEGRANDS[integrand], dims, n, _ACCUM[accum],
                               C.byref(row), _stream(stream)))
    return {"n": row.n, "estimate": row.estimate, "abs_error": row.abs_error,
            "seconds": row.seconds}


def integrate_partials(kind: str, integrand: str, n: int, dims: int, chunk_begin: int,
                       chunk_end: int, accum: str = "kahan", *, stream_dims: Optional[int] = None,
                       generator=None, matrices: Optional[GeneratorMatrixSet] = None,
                       sobol_scrambles=None, scramble: str = "plain", linear_factors=None,
                       pixel=(0, 0), order: int = 1, spp: int = 1, width: int = 0,
                       height: int = 0, xor_seed: int = 0, xor_point_count: int = 1, stream=None):
    """The integration restricted to 4096-index chunks [chunk_begin, chunk_end)
    of [0, n): a float64 array of the chunks' Kahan partials (kahan) or the
    exact int64 sum of llround(f * 2^32) (int). Rank shares of a multi-GPU
    integrate (paper_2307_15584_b200.distributed.integrate_distributed)."""
    k = sampler_kind_from_name(kind)
    if accum not in _ACCUM:
        raise ConfigError("accumulation mode must be 'kahan' or 'int'")
    if integrand not in _INTEGRANDS:
        raise ConfigError("unknown integrand: " + integrand)
    sd = dims if stream_dims is None else stream_dims
    p, keep = _stream_params(sd, generator, matrices, sobol_scrambles, scramble, linear_factors,
                             pixel, order, spp, width, height, xor_seed, xor_point_count)
    parts = np.zeros(max(chunk_end - chunk_begin, 1), np.float64)
    isum = C.c_int64(0)
    _check(lib().qmc_integrate_partials(k, C.byref(p), _INTEGRANDS[integrand], dims, n,
                                        chunk_begin, chunk_end, _ACCUM[accum], parts.ctypes.data,
                                        C.byref(isum), _stream(stream)))
    return parts[:chunk_end - chunk_begin] if accum == "kahan" else isum.value


def reduce_deterministic(ranks, values) -> float:
    """reduce_deterministic (quality.cpp:158-166): CompensatedSum in rank order."""
    r = np.ascontiguousarray(ranks, dtype=np.uint64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if r.size != v.size:
        raise ValueError("ranks and values differ in length")
    out = f64()
    _check(lib().qmc_reduce_deterministic(r.ctypes.data, v.ctypes.data, r.size, C.byref(out)))
    return out.value


def render(width: int, height: int, spp: int = 1, kind: str = "pixel-shifted-lattice",
           accum: str = "kahan", seed: int = 0, generator=None,
           matrices: Optional[GeneratorMatrixSet] = None, tables: Optional[XorTables] = None,
           rows=None, out=None, stream=None):
    """render(RenderJob) (render.cpp:83-143) for rows [r0, r1) of the image.

    Returns a [rows, width] float32 tensor (or fills `out`, device or host)."""
    if accum not in _ACCUM:
        raise ConfigError("accumulation mode must be 'kahan' or 'int'")
    job = RenderJob()
    job.width, job.height, job.spp = width, height, spp
    job.kind = sampler_kind_from_name(kind)
    job.accum = _ACCUM[accum]
    job.seed = seed
    keep = None
    if generator is not None:
        keep = _u32_host(generator)
        job.generator, job.generator_dims = keep.ctypes.data, keep.size
    if matrices is not None:
        job.matrices = matrices.handle
    if tables is not None:
        job.tables = tables.handle
    r0, r1 = rows if rows is not None else (0, height)
    if out is None:
        torch = _torch()
        out = torch.empty((max(r1 - r0, 0), width), dtype=torch.float32, device="cuda")
    _check_out(out, max(r1 - r0, 0) * width, "float32")
    _check(lib().qmc_render(C.byref(job), r0, r1, _ptr(out), _stream(stream)))
    return out


def _render_job(width, height, spp, kind, accum, seed, generator, matrices, tables):
    if accum not in _ACCUM:
        raise ConfigError("accumulation mode must be 'kahan' or 'int'")
    job = RenderJob()
    job.width, job.height, job.spp = width, height, spp
    job.kind = sampler_kind_from_name(kind)
    job.accum = _ACCUM[accum]
    job.seed = seed
    keep = []
    if generator is not None:
        g = _u32_host(generator)
        keep.append(g)
        job.generator, job.generator_dims = g.ctypes.data, g.size
    if matrices is not None:
        job.matrices = matrices.handle
    if tables is not None:
        job.tables = tables.handle
    return job, keep


def render_devices(width: int, height: int, spp: int, devices, kind: str = "pixel-shifted-lattice",
                   accum: str = "kahan", seed: int = 0, generator=None,
                   matrices: Optional[GeneratorMatrixSet] = None,
                   tables: Optional[XorTables] = None, out=None) -> np.ndarray:
    """render(RenderJob) across the GPUs `devices` of this process (row bands,
    one host thread per device; qmc_render_devices). Returns a host
    [height, width] float32 array, bit-identical to a one-device render."""
    job, keep = _render_job(width, height, spp, kind, accum, seed, generator, matrices, tables)
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    if out is None:
        out = np.empty((height, width), np.float32)
    _check_out(out, height * width, "float32")
    _check(lib().qmc_render_devices(C.byref(job), devs.ctypes.data, devs.size, _ptr(out)))
    return out


def render_samples_devices(width: int, height: int, spp: int, devices,
                           kind: str = "pixel-shifted-lattice", seed: int = 0, generator=None,
                           matrices: Optional[GeneratorMatrixSet] = None,
                           tables: Optional[XorTables] = None, out=None) -> np.ndarray:
    """The paper's sample partition over `devices` (a power-of-two count) with
    the int64 reduction fused into the render kernels (atomic adds into one
    accumulator on devices[0], peer access across GPUs). Returns the host
    [height, width] image, bit-identical to render(..., accum="int")."""
    job, keep = _render_job(width, height, spp, kind, "int", seed, generator, matrices, tables)
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    if out is None:
        out = np.empty((height, width), np.float32)
    _check_out(out, height * width, "float32")
    _check(lib().qmc_render_samples_devices(C.byref(job), devs.ctypes.data, devs.size,
                                            _ptr(out)))
    return out


def render_partial(width: int, height: int, spp: int, part: int, parts: int,
                   kind: str = "pixel-shifted-lattice", seed: int = 0, generator=None,
                   matrices: Optional[GeneratorMatrixSet] = None,
                   tables: Optional[XorTables] = None, rows=None, out=None, stream=None):
    """Int-mode partial render over the samples of part `part` of `parts`
    (i == rev_2(part) mod parts): int64 [rows, width] accumulators."""
    job, keep = _render_job(width, height, spp, kind, "int", seed, generator, matrices, tables)
    r0, r1 = rows if rows is not None else (0, height)
    if out is None:
        torch = _torch()
        out = torch.empty((max(r1 - r0, 0), width), dtype=torch.int64, device="cuda")
    _check_out(out, max(r1 - r0, 0) * width, "int64")
    _check(lib().qmc_render_partial(C.byref(job), part, parts, r0, r1, _ptr(out),
                                    _stream(stream)))
    return out


def render_finalize(acc, spp: int, out=None, stream=None):
    """float(sum / 2^32 / spp) of summed partial accumulators."""
    torch = _torch()
    if out is None:
        out = torch.empty(acc.shape, dtype=torch.float32, device=acc.device)
    _check_out(acc, acc.numel(), "int64")
    _check_out(out, acc.numel(), "float32")
    _check(lib().qmc_render_finalize(_ptr(acc), acc.numel(), spp, _ptr(out), _stream(stream)))
    return out


def load_generator_vector(text: str) -> list:
    """load_generator_vector (lattice.cpp:21-46)."""
    n = u32()
    _check(lib().qmc_load_generator_vector(text.encode(), None, 0, C.byref(n)))
    out = np.zeros(n.value, np.uint32)
    _check(lib().qmc_load_generator_vector(text.encode(), out.ctypes.data, n.value, C.byref(n)))
    return out.tolist()


def load_linear_factors(text: str, dims: int) -> list:
    """load_linear_factors (radical.cpp:281-306)."""
    out = np.zeros(max(dims, 1), np.uint32)
    _check(lib().qmc_load_linear_factors(text.encode(), dims, out.ctypes.data))
    return out[:dims].tolist()


def fnv1a64(data) -> int:
    """fnv1a64 (image.cpp:54-63) of bytes or an array's bytes."""
    buf = np.ascontiguousarray(np.frombuffer(data, np.uint8) if isinstance(data, (bytes, bytearray))
                               else data)
    return lib().qmc_fnv1a64(buf.ctypes.data, buf.nbytes)


def write_points_csv(points, stream=None) -> bytes:
    """`qmckit points --format csv` text of an [n, dims] float array."""
    if isinstance(points, np.ndarray):
        points = np.ascontiguousarray(points, dtype=np.float32)
    n, dims = points.shape
    ln = C.c_size_t(0)
    _check(lib().qmc_write_points_csv(_ptr(points), n, dims, None, C.byref(ln), _stream(stream)))
    buf = C.create_string_buffer(max(ln.value, 1))
    _check(lib().qmc_write_points_csv(_ptr(points), n, dims, buf, C.byref(ln), _stream(stream)))
    return buf.raw[: ln.value]


def write_pnm(image, channels: int = 1, stream=None) -> bytes:
    """write_pgm (channels=1) / write_ppm (channels=3) of an [h, w] float image."""
    if isinstance(image, np.ndarray):
        image = np.ascontiguousarray(image, dtype=np.float32)
    h, w = image.shape
    n = C.c_size_t(0)
    _check(lib().qmc_write_pnm(_ptr(image), w, h, channels, None, C.byref(n), _stream(stream)))
    buf = C.create_string_buffer(n.value)
    _check(lib().qmc_write_pnm(_ptr(image), w, h, channels, buf, C.byref(n), _stream(stream)))
    return buf.raw[: n.value]


def scene_value(xy, out=None, stream=None):
    """Device scene_value (render.cpp:17-26) for an [n, 2] float64 array."""
    if isinstance(xy, np.ndarray):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.empty(xy.shape[0], np.float64) if out is None else out
    else:
        torch = _torch()
        out = torch.empty(xy.shape[0], dtype=torch.float64, device=xy.device) if out is None else out
    _check(lib().qmc_scene_value(_ptr(xy), _ptr(out), xy.shape[0], _stream(stream)))
    return out


def run_bench_kernel(kernel: str, count: int, dims: int, stream=None) -> dict:
    """run_bench_kernel (bench.cpp:79-150) on the device: the BenchResult
    fields; `checksum` equals the reference's for the same arguments."""
    r = BenchResult()
    _check(lib().qmc_run_bench_kernel(kernel.encode(), count, dims, C.byref(r), _stream(stream)))
    return {"kernel": kernel, "evaluations": r.evaluations, "seconds": r.seconds,
            "components_per_second": r.components_per_second, "checksum": r.checksum}


def fp64_probe(iters: int = 4096, stream=None) -> float:
    """Measured dense FP64 FMA throughput of the current GPU, flop/s."""
    v = f64()
    _check(lib().qmc_fp64_probe(iters, C.byref(v), _stream(stream)))
    return v.value


# ------------------------------------------------ multi-GPU render over NCCL
_PARTITION = {"rows": 0, "samples": 1}


def _prefer_process_nccl() -> None:
    """Point the library's lazy NCCL load at the copy PyTorch uses (the
    nvidia-nccl wheel), so one process never maps two NCCL builds; an explicit
    QMC_NCCL_LIBRARY wins."""
    if os.environ.get("QMC_NCCL_LIBRARY"):
        return
    try:
        import nvidia.nccl as nn

        for base in nn.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["QMC_NCCL_LIBRARY"] = cand
                return
    except ImportError:
        pass


def nccl_version() -> int:
    """NCCL_VERSION_CODE of the NCCL the library bound (e.g. 22809)."""
    _prefer_process_nccl()
    v = i32()
    _check(lib().qmc_nccl_version(C.byref(v)))
    return v.value


class Comm:
    """An NCCL communicator owned by libqmcgpu (qmc_comm)."""

    def __init__(self, handle: int):
        self._h = handle

    @staticmethod
    def unique_id() -> bytes:
        """ncclGetUniqueId (rank 0), to ship to the other ranks."""
        _prefer_process_nccl()
        buf = C.create_string_buffer(128)
        _check(lib().qmc_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def init_rank(cls, uid: bytes, nranks: int, rank: int) -> "Comm":
        """ncclCommInitRank on the current CUDA device."""
        _prefer_process_nccl()
        if len(uid) != 128:
            raise ValueError("unique id must be 128 bytes")
        h = P()
        _check(lib().qmc_comm_init_rank(C.c_char_p(uid), nranks, rank, C.byref(h)))
        return cls(h.value)

    @classmethod
    def init_all(cls, devices) -> list:
        """ncclCommInitAll: one communicator per device of this process."""
        _prefer_process_nccl()
        devs = np.ascontiguousarray(devices, dtype=np.int32)
        hs = (P * max(devs.size, 1))()
        _check(lib().qmc_comm_init_all(devs.ctypes.data, devs.size, hs))
        return [cls(hs[k]) for k in range(devs.size)]

    @classmethod
    def from_torch_group(cls, group=None) -> "Comm":
        """A library communicator spanning the ranks of a torch.distributed
        group: rank 0's unique id travels over the group, then every rank
        calls ncclCommInitRank on its current device."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.init_rank(obj[0], world, rank)

    def info(self):
        r, n, d = i32(), i32(), i32()
        _check(lib().qmc_comm_info(self._h, C.byref(r), C.byref(n), C.byref(d)))
        return {"rank": r.value, "nranks": n.value, "device": d.value}

    @property
    def handle(self) -> int:
        return self._h

    def destroy(self) -> None:
        if self._h:
            lib().qmc_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:  # pragma: no cover - interpreter teardown
            pass


def render_nccl(width: int, height: int, spp: int, comm: Comm, mode: str = "rows",
                kind: str = "pixel-shifted-lattice", accum: str = "kahan", seed: int = 0,
                generator=None, matrices: Optional[GeneratorMatrixSet] = None,
                tables: Optional[XorTables] = None, out=None, stream=None):
    """render(RenderJob) by every rank of `comm` (qmc_render_nccl): row bands +
    ncclAllGather ("rows") or the paper's sample partition + int64
    ncclAllReduce ("samples", int accumulator). Every rank gets the whole
    [height, width] float32 image on its device."""
    if mode not in _PARTITION:
        raise ValueError("mode must be 'rows' or 'samples'")
    job, keep = _render_job(width, height, spp, kind, accum, seed, generator, matrices, tables)
    if out is None:
        torch = _torch()
        out = torch.empty((height, width), dtype=torch.float32, device="cuda")
    _check_out(out, height * width, "float32")
    _check(lib().qmc_render_nccl(C.byref(job), comm.handle, _PARTITION[mode], _ptr(out),
                                 _stream(stream)))
    return out


def render_nccl_devices(width: int, height: int, spp: int, devices, mode: str = "rows",
                        kind: str = "pixel-shifted-lattice", accum: str = "kahan", seed: int = 0,
                        generator=None, matrices: Optional[GeneratorMatrixSet] = None,
                        tables: Optional[XorTables] = None, out=None) -> np.ndarray:
    """The NCCL render across distinct `devices` of this process
    (qmc_render_nccl_devices); returns the host [height, width] image."""
    if mode not in _PARTITION:
        raise ValueError("mode must be 'rows' or 'samples'")
    _prefer_process_nccl()
    job, keep = _render_job(width, height, spp, kind, accum, seed, generator, matrices, tables)
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    if out is None:
        out = np.empty((height, width), np.float32)
    _check_out(out, height * width, "float32")
    _check(lib().qmc_render_nccl_devices(C.byref(job), devs.ctypes.data, devs.size,
                                         _PARTITION[mode], _ptr(out)))
    return out
