"""ctypes binding of the C ABI in include/detlsh_b200.h.

The shared library is built in-tree (``make -C paper_2406_10938_b200``) and is
the only compute path: there is no CPU fallback.  Loading fails loudly if the
library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libdetlsh_b200.so")
HEADER = os.path.join(ROOT, "include", "detlsh_b200.h")

DETLSH_OK = 0
DETLSH_E_INVALID = 1
DETLSH_E_CUDA = 2
DETLSH_E_FORMAT = 3

F_DEVICE_PTRS = 0x1
F_SAMPLE_GPU = 0x2
F_BORROW_DATA = 0x4
F_NO_CODES = 0x8
F_NO_U8 = 0x10
F_NO_TC = 0x20
F_PAA = 0x40
RANGE_EXACT = 0x100


class Params(C.Structure):
    """detlsh_params == detlsh::LshParams field order (projection.hpp:79-92)."""

    _fields_ = [
        ("K", C.c_int32), ("L", C.c_int32), ("c", C.c_double), ("beta", C.c_double),
        ("epsilon", C.c_double), ("alpha1", C.c_double), ("alpha2", C.c_double),
        ("n_regions", C.c_int32), ("sample_fraction", C.c_double),
        ("leaf_capacity", C.c_int32), ("r_min", C.c_double), ("k", C.c_int32),
    ]


class FormatError(RuntimeError):
    """detlsh::FormatError (errors.hpp:19-28)."""


_lib = None


def header_symbols() -> list[str]:
    """Every function the C header declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(detlsh_[a-z0-9_]+)\s*\(", text)))


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, u64, i32, dbl, u32 = C.c_void_p, C.c_uint64, C.c_int32, C.c_double, C.c_uint32
    P = C.POINTER(Params)
    sig = {
        "detlsh_candidate_budget": ([dbl, u64, i32], u64),
        "detlsh_derive_params": ([i32, dbl, i32, vp], C.c_int),
        "detlsh_sample_hash_family": ([i32, i32, i32, u64, vp], C.c_int),
        "detlsh_chi2_cdf": ([dbl, i32], dbl),
        "detlsh_chi2_quantile": ([dbl, i32], dbl),
        "detlsh_device_count": ([], C.c_int),
        "detlsh_gpu_last_error": ([], C.c_char_p),
        "detlsh_version": ([], C.c_char_p),
        "detlsh_select_row_breakpoints": ([vp, u64, i32, u64, vp, C.POINTER(u64)], C.c_int),
        "detlsh_launch_count": ([], u64),
        "detlsh_query_phase_cycles": ([vp], None),
        "detlsh_test_tc_gemm_u8": ([vp, vp, i32, i32, vp], C.c_int),
        "detlsh_profile_enable": ([i32], None),
        "detlsh_profile_collect": ([C.c_char_p, i32, vp, vp, i32], C.c_int),
        "detlsh_gpu_build": ([vp, u64, i32, P, u64, i32, u32, C.POINTER(vp)], C.c_int),
        "detlsh_gpu_build_with_family": ([vp, u64, i32, P, vp, i32, i32, u64, u64, i32, u32,
                                          C.POINTER(vp)], C.c_int),
        "detlsh_gpu_free": ([vp], None),
        "detlsh_gpu_query": ([vp, vp, u64, i32, u32, vp, vp, vp, vp, vp, vp], C.c_int),
        "detlsh_gpu_query_check": ([vp, vp], C.c_int),
        "detlsh_gpu_estimate_rmin": ([vp, vp, u64, i32, u32, C.POINTER(dbl)], C.c_int),
        "detlsh_gpu_project_query": ([vp, vp, u64, vp, u32], C.c_int),
        "detlsh_gpu_range_query": ([vp, i32, vp, u64, vp, u64, u32, vp, u64, vp], C.c_int),
        "detlsh_gpu_synth": ([i32, u64, u64, u64, i32, vp, i32, vp], C.c_int),
        "detlsh_gpu_rc_ann": ([vp, vp, u64, dbl, dbl, u32, vp, vp, vp, vp, vp], C.c_int),
        "detlsh_gpu_brute_force_knn": ([vp, u64, i32, vp, u64, i32, vp, u32, vp, vp, i32, vp], C.c_int),
        "detlsh_vectors_shape": ([C.c_char_p, C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)], C.c_int),
        "detlsh_gpu_read_vectors": ([C.c_char_p, vp, u64, i32, i32, vp], C.c_int),
        "detlsh_gpu_merge_topk": ([vp, vp, vp, i32, u64, i32, vp, vp, vp, vp], C.c_int),
        "detlsh_gpu_sharded_build": ([vp, u64, i32, P, u64, vp, i32, u32, C.POINTER(vp)], C.c_int),
        "detlsh_gpu_sharded_query": ([vp, vp, u64, i32, u32, vp, vp, vp, vp], C.c_int),
        "detlsh_gpu_sharded_count": ([vp], i32),
        "detlsh_gpu_sharded_shard": ([vp, i32, C.POINTER(u64), C.POINTER(u64)], vp),
        "detlsh_gpu_sharded_free": ([vp], None),
        "detlsh_gpu_get_params": ([vp, P], C.c_int),
        "detlsh_gpu_n": ([vp], u64),
        "detlsh_gpu_d": ([vp], i32),
        "detlsh_gpu_sample_size": ([vp], u64),
        "detlsh_gpu_family_seed": ([vp], u64),
        "detlsh_gpu_has_family": ([vp], i32),
        "detlsh_gpu_row_u8": ([vp], i32),
        "detlsh_gpu_export_family": ([vp, vp], C.c_int),
        "detlsh_gpu_export_table": ([vp, vp], C.c_int),
        "detlsh_gpu_export_codes": ([vp, vp], C.c_int),
        "detlsh_gpu_tree_num_nodes": ([vp, i32, C.POINTER(u64)], C.c_int),
        "detlsh_gpu_export_tree": ([vp, i32] + [vp] * 10, C.c_int),
        "detlsh_gpu_build_timings": ([vp, vp, i32, C.c_char_p, i32], C.c_int),
        "detlsh_gpu_save_detl": ([vp, vp, u64, C.POINTER(u64)], C.c_int),
        "detlsh_gpu_project": ([vp, i32, i32, vp, u64, i32, vp, i32, u32], C.c_int),
        "detlsh_gpu_select_breakpoints": ([vp, u64, i32, i32, i32, dbl, u64, vp, C.POINTER(u64),
                                           i32, u32], C.c_int),
        "detlsh_gpu_encode": ([vp, u64, i32, i32, vp, i32, vp, i32, u32], C.c_int),
        "detlsh_gpu_build_tree": ([vp, u64, i32, i32, i32, i32, i32, i32, u32, C.POINTER(vp)],
                                  C.c_int),
        "detlsh_gpu_tree_nodes": ([vp, C.POINTER(u64)], C.c_int),
        "detlsh_gpu_tree_export": ([vp] + [vp] * 10, C.c_int),
        "detlsh_gpu_tree_free": ([vp], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code onto the reference's exception taxonomy."""
    if rc == DETLSH_OK:
        return
    msg = load().detlsh_gpu_last_error().decode(errors="replace")
    if rc == DETLSH_E_INVALID:
        raise ValueError(msg)  # std::invalid_argument
    if rc == DETLSH_E_FORMAT:
        raise FormatError(msg)
    raise RuntimeError(msg)
