"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the two CPU checkers.

* ``load_oracle()`` -> the C restatement ``oracle/libqmc_oracle.so``
  (``qmc_oracle.c``; each function cites the reference file:line it follows).
* ``load_ref()``    -> the unmodified reference library compiled from
  ``/root/reference/proj/src`` plus our extern "C" shim
  (``oracle/_ref/libqmcref.so``, built by ``oracle/Makefile``).

Only ``tests/``, ``bench.py`` (cpu_baseline and ``--impl reference``) and
``__graft_entry__.smoke()`` may import this package, and only as the checker or
the timed CPU baseline. The product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libqmc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqmcref.so")

u32, u64, i32, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_double
P = C.c_void_p
pu32, pu64 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
cstr = C.c_char_p


def build() -> None:
    """Compile the oracle (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


_oracle = None
_ref = None


def load_oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        _sig(lib, "qo_clz32", u32, u32)
        _sig(lib, "qo_brev32", u32, u32)
        _sig(lib, "qo_map_bits", u32, u32)
        _sig(lib, "qo_map_range", None, u32, u64, P)
        _sig(lib, "qo_prime", i32, u32, pu32)
        _sig(lib, "qo_prime_max_power", i32, u32, pu32)
        _sig(lib, "qo_max_power_fitting_u32", u32, u32)
        _sig(lib, "qo_radical_inverse_fixed", u32, u32, u32)
        _sig(lib, "qo_radical_inverse_linscramble_fixed", u32, u32, u32, u32)
        _sig(lib, "qo_radical_inverse_permuted_fixed", u32, u32, u32, P)
        _sig(lib, "qo_faure_permutation", None, u32, P)
        _sig(lib, "qo_tensor_digit_table", u32, P, u32, u32, P)
        _sig(lib, "qo_radical_inverse_tabled_fixed", u32, u32, u32, u32, P, P)
        _sig(lib, "qo_build_matrices", None, u32, P, P, P, P)
        _sig(lib, "qo_sobol_component_fixed", u32, u64, P, u32)
        _sig(lib, "qo_sobol_fill_fixed", None, u64, u64, u32, P, P, P)
        _sig(lib, "qo_sobol_fill_f32", None, u64, u64, u32, P, P, P)
        _sig(lib, "qo_owen_scramble", u32, u32, u32)
        _sig(lib, "qo_sobol_owen_fill_fixed", None, u64, u64, u32, P, P, P)
        _sig(lib, "qo_lattice_component_fixed", u32, u32, u32)
        _sig(lib, "qo_lattice_cp_fixed", u32, u32, u32, u32)
        _sig(lib, "qo_pixel_hash", u32, u32, u32, u32)
        _sig(lib, "qo_random_lattice_component_fixed", u32, u32, u32, u32, u32)
        _sig(lib, "qo_lfsr_generator_vector", i32, u32, u32, P)
        _sig(lib, "qo_lattice_shift_fixed", i32, u32, u32, P, u32, P)
        _sig(lib, "qo_hilbert_index", i32, u32, u32, u32, pu64)
        _sig(lib, "qo_hilbert_xy", i32, u64, u32, pu32, pu32)
        _sig(lib, "qo_hilbert_phi3_fixed", u32, u32, u32, u32)
        _sig(lib, "qo_digit_reverse", u64, u64, u32, u32)
        _sig(lib, "qo_halton_enum_init", i32, u32, u32, P)
        _sig(lib, "qo_halton_enum_offset", u64, P, u32, u32)
        _sig(lib, "qo_partition", i32, u32, u32, u32, pu64, pu64)
        _sig(lib, "qo_scene_value", f64, f64, f64)
        _sig(lib, "qo_hilbert_order_for", u32, u32, u32)
        _sig(lib, "qo_render", i32, u32, u32, u32, i32, i32, u32, P, P)
        _sig(lib, "qo_fnv1a64", u64, P, u64)
        _sig(lib, "qo_render_partial_int", i32, u32, u32, u32, i32, u32, P, u32, u32, P)
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        lib = C.CDLL(REF_SO)
        _sig(lib, "ref_last_error", cstr)
        _sig(lib, "ref_map_bits", u32, u32)
        _sig(lib, "ref_map_bulk", None, P, P, u64)
        _sig(lib, "ref_map_range", None, u32, u64, P)
        _sig(lib, "ref_bit_reverse32", u32, u32)
        _sig(lib, "ref_clz32", u32, u32)
        _sig(lib, "ref_prime", i32, u32, pu32)
        _sig(lib, "ref_prime_max_power", i32, u32, pu32)
        _sig(lib, "ref_radical_fixed_fill", i32, u32, u64, u32, i32, u32, P)
        _sig(lib, "ref_radical_tabled_fixed_fill", i32, u32, u64, i32, P)
        _sig(lib, "ref_faure_permutation", i32, u32, P)
        _sig(lib, "ref_tensor_table", i32, P, u32, u32, P, pu32)
        _sig(lib, "ref_tabled_halton_fixed_fill", i32, u32, u64, u32, P)
        _sig(lib, "ref_build_matrices_builtin", i32, u32, P)
        _sig(lib, "ref_build_matrices_text", i32, cstr, u32, P)
        _sig(lib, "ref_sobol_fixed_fill", i32, u64, u64, u32, P, P, i32)
        _sig(lib, "ref_sobol_fill", i32, u64, u64, u32, P, P, i32)
        _sig(lib, "ref_pixel_hash", u32, u32, u32, u32)
        _sig(lib, "ref_lfsr_generator_vector", i32, u32, u32, P)
        _sig(lib, "ref_lattice_fill", i32, u64, u64, u32, P, P, P, i32)
        _sig(lib, "ref_lattice_shift_fixed", i32, u32, u32, P, u32, P)
        _sig(lib, "ref_hilbert_index", i32, u32, u32, u32, pu64)
        _sig(lib, "ref_hilbert_xy", i32, u64, u32, pu32, pu32)
        _sig(lib, "ref_hilbert_phi3_fixed", i32, u32, u32, u32, pu32)
        _sig(lib, "ref_halton_pixel_enum", i32, u32, u32, u32, u32, pu64, pu64, P)
        _sig(lib, "ref_digit_reverse", u64, u64, u32, u32)
        _sig(lib, "ref_partition", i32, u32, u32, u32, pu64, pu64)
        _sig(lib, "ref_stream_fill", i32, cstr, u32, u32, cstr, u32, u32, u32, u32, u32, u32,
             u64, u64, P)
        _sig(lib, "ref_render", i32, u32, u32, u32, cstr, cstr, u32, u32, P)
        _sig(lib, "ref_scene_value", f64, f64, f64)
        _sig(lib, "ref_hilbert_order_for", u32, u32, u32)
        _sig(lib, "ref_fnv1a64", u64, P, u64)
        _sig(lib, "ref_run_bench_kernel", i32, cstr, u64, u32, C.POINTER(f64), pu64)
        _sig(lib, "ref_integrate", i32, cstr, u32, u32, cstr, u64, cstr, u32, C.POINTER(f64))
        _sig(lib, "ref_integrate_sobol_text", i32, cstr, u32, cstr, u64, cstr, u32, C.POINTER(f64))
        _sig(lib, "ref_radical_fill", i32, u64, u64, u32, P, i32)
        _sig(lib, "ref_halton_linear_fill", i32, u64, u64, u32, P, i32)
        _sig(lib, "ref_neumaier", f64, P, u64)
        _sig(lib, "ref_reduce_deterministic", f64, P, P, u64)
        _sig(lib, "ref_l2_star", i32, P, u64, u32, C.POINTER(f64))
        _sig(lib, "ref_min_toroidal", i32, P, u64, u32, C.POINTER(f64))
        _sig(lib, "ref_stratification", i32, cstr, u32, u32, u32, u32, C.POINTER(i32))
        _sig(lib, "ref_white_noise_xor_file", i32, u32, u32, u32, P, pu64)
        _sig(lib, "ref_load_generator_vector", i32, cstr, P, u32, pu32)
        _sig(lib, "ref_load_linear_factors", i32, cstr, u32, P)
        _sig(lib, "ref_write_pnm", i32, P, u32, u32, i32, P, pu64)
        _sig(lib, "ref_xor_stream_fill", i32, P, u64, u32, u32, u32, u32, u32, u64, u64, P)
        _ref = lib
    return _ref


def ptr(a) -> int:
    """Address of a numpy array (or None -> NULL)."""
    return None if a is None else a.ctypes.data
