"""ctypes mirror of include/bfla.h — argument marshalling only.

Every entry point of the C ABI is exposed under the same name.  Tensors are passed as raw device
pointers (torch is used for memory and streams only); every step of the path runs in
libbfla.so's CUDA kernels.  There is no fallback: if the library is missing or a call returns a
non-OK status, a RuntimeError is raised.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbfla.so")


def use_variant(name: str) -> None:
    """Tools and debug tests only: load libbfla_<name>.so (build.py variants: debug, exp, trace, or an
    A/B build of tools/ab_build.py) instead of the product library.  Must precede the first lib()."""
    global LIB_PATH
    path = os.path.join(_HERE, f"libbfla_{name}.so") if name else os.path.join(_HERE, "libbfla.so")
    if _lib is not None and path != LIB_PATH:
        raise RuntimeError(f"{LIB_PATH} is already loaded")
    LIB_PATH = path

BFLA_OK = 0
STATUS = {0: "BFLA_OK", 1: "BFLA_ERR_INVALID_ARGUMENT", 2: "BFLA_ERR_UNSUPPORTED", 3: "BFLA_ERR_MISALIGNED",
          4: "BFLA_ERR_WORKSPACE", 5: "BFLA_ERR_CAPACITY", 6: "BFLA_ERR_CUDA"}
KV_CONTIGUOUS, KV_PAGED = 0, 1
POOL_FLATTEN, POOL_MEAN = 0, 1
SELECT_MASS, SELECT_RATIO = 0, 1
SCORES_AUTO, SCORES_CANONICAL = 0, 1
MASK_PER_KV_HEAD, MASK_PER_Q_HEAD = 0, 1

i32, i64, f32, u64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_uint64, ctypes.c_void_p


class bfla_problem(ctypes.Structure):
    _fields_ = [("batch", i32), ("h_q", i32), ("h_kv", i32), ("head_dim", i32),
                ("n_q", i32), ("n_kv", i32), ("softmax_scale", f32), ("head_offset", i32),
                ("q", vp), ("q_stride", i64 * 3), ("o", vp), ("o_stride", i64 * 3), ("lse", vp),
                ("kv_layout", i32), ("k", vp), ("v", vp), ("kv_stride", i64 * 3),
                ("page_size", i32), ("num_pages", i32), ("max_pages_per_seq", i32), ("page_table", vp),
                ("seqlens", vp)]


class bfla_config(ctypes.Structure):
    _fields_ = [("block_b", i32), ("group_g", i32), ("tile_t", i32), ("pool", i32), ("select", i32),
                ("gamma", f32), ("keep_ratio", f32), ("n_sink", i32), ("n_local", i32), ("eta", i32),
                ("rho", f32), ("seed", u64), ("scores_path", i32), ("mask_groups", i32),
                ("certify_slack", f32)]


class bfla_stats(ctypes.Structure):
    _fields_ = [("causal_tiles", u64), ("kept_tiles", u64), ("label", u64 * 6), ("rows", u64),
                ("rows_exact_tie", u64), ("blocks_kept", u64), ("rows_flagged", u64), ("rows_recomputed", u64),
                ("reserved", u64 * 3)]


class bfla_mask(ctypes.Structure):
    _fields_ = [("coarse_bits", vp), ("tile_bits", vp), ("tile_list", vp), ("tile_list_capacity", i64),
                ("tile_count", vp), ("tile_label", vp), ("kept_mass", vp), ("stats", vp)]


MAX_MIRRORS = 7


class bfla_mirrors(ctypes.Structure):
    _fields_ = [("n", i32), ("o", vp * MAX_MIRRORS), ("lse", vp * MAX_MIRRORS), ("multicast_o", vp),
                ("multicast_lse", vp)]


MAX_PARTS = 8


class bfla_partials(ctypes.Structure):
    _fields_ = [("n", i32), ("o", vp * MAX_PARTS), ("lse", vp * MAX_PARTS)]


_lib = None

ENTRY_POINTS = ["bfla_workspace_size", "bfla_tile_list_capacity", "bfla_block_mask", "bfla_expand_rescue",
                "bfla_sparse_prefill", "bfla_sparse_prefill_rows", "bfla_sparse_prefill_mirrored",
                "bfla_sparse_prefill_kvrange", "bfla_merge_partials",
                "bfla_balance_rows", "bfla_prefill",
                "bfla_status_string", "bfla_last_error",
                "bfla_kernel_launches"]


def lib():
    """Load libbfla.so (raises if it is missing — no CPU or eager fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libbfla.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        L.bfla_workspace_size.argtypes = [P(bfla_problem), P(bfla_config)]
        L.bfla_workspace_size.restype = ctypes.c_size_t
        L.bfla_tile_list_capacity.argtypes = [P(bfla_problem), P(bfla_config)]
        L.bfla_tile_list_capacity.restype = i64
        for name, mask_t in [("bfla_block_mask", P(bfla_mask)), ("bfla_expand_rescue", P(bfla_mask)),
                             ("bfla_sparse_prefill", P(bfla_mask)), ("bfla_prefill", P(bfla_mask))]:
            fn = getattr(L, name)
            fn.argtypes = [P(bfla_problem), P(bfla_config), mask_t, vp, ctypes.c_size_t, vp]
            fn.restype = ctypes.c_int
        L.bfla_sparse_prefill_rows.argtypes = [P(bfla_problem), P(bfla_config), P(bfla_mask), i64, i64, vp,
                                               ctypes.c_size_t, vp]
        L.bfla_sparse_prefill_rows.restype = ctypes.c_int
        L.bfla_sparse_prefill_mirrored.argtypes = [P(bfla_problem), P(bfla_config), P(bfla_mask), i64, i64,
                                                   P(bfla_mirrors), vp, ctypes.c_size_t, vp]
        L.bfla_sparse_prefill_mirrored.restype = ctypes.c_int
        L.bfla_sparse_prefill_kvrange.argtypes = [P(bfla_problem), P(bfla_config), P(bfla_mask), i64, i64, i64, i64,
                                                  vp, ctypes.c_size_t, vp]
        L.bfla_sparse_prefill_kvrange.restype = ctypes.c_int
        L.bfla_merge_partials.argtypes = [P(bfla_problem), P(bfla_partials), vp]
        L.bfla_merge_partials.restype = ctypes.c_int
        L.bfla_balance_rows.argtypes = [P(i32), i32, i32, i32, i32, i32, P(i64)]
        L.bfla_balance_rows.restype = ctypes.c_int
        L.bfla_status_string.argtypes = [ctypes.c_int]
        L.bfla_status_string.restype = ctypes.c_char_p
        L.bfla_last_error.argtypes = []
        L.bfla_last_error.restype = ctypes.c_char_p
        L.bfla_kernel_launches.argtypes = []
        L.bfla_kernel_launches.restype = u64
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != BFLA_OK:
        detail = lib().bfla_last_error().decode()
        raise RuntimeError(f"{what}: {STATUS.get(status, status)}: {detail}")
