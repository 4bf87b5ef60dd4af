"""ctypes binding of libalto_b200.so (the C ABI declared in include/alto_b200.h).

The shared library is built in-tree by `make` (or __graft_entry__.build()).
There is no CPU fallback: if the library or a CUDA device is missing, the
device entry points raise `RuntimeError` loudly.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_int32, c_int64,
                    c_size_t, c_uint8, c_void_p)

import numpy as np

ALTO_MAX_ORDER = 8
ALTO_OK, ALTO_EINVAL, ALTO_ECUDA, ALTO_EUNSUPPORTED, ALTO_ENCCL, ALTO_ESINGULAR = range(6)
ALTO_F32, ALTO_F64, ALTO_I64 = 0, 1, 2

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libalto_b200.so")


class CLayout(Structure):
    _fields_ = [
        ("order", c_int32),
        ("n_words", c_int32),
        ("total_bits", c_int32),
        ("width", c_int32),
        ("dims", c_int64 * ALTO_MAX_ORDER),
        ("bits", c_int32 * ALTO_MAX_ORDER),
        ("pos", (c_uint8 * 64) * ALTO_MAX_ORDER),
    ]


class CMttkrpArgs(Structure):
    _fields_ = [
        ("lay", POINTER(CLayout)),
        ("d_tables", c_void_p),
        ("keys", c_void_p),
        ("values", c_void_p),
        ("m", c_int64),
        ("mode", c_int32),
        ("rank", c_int32),
        ("value_dtype", c_int32),
        ("factor_dtype", c_int32),
        ("factors", c_void_p * ALTO_MAX_ORDER),
        ("out", c_void_p),
        ("out_dtype", c_int32),
        ("tile", c_int32),
        ("zero_out", c_int32),
        ("hot_slot", c_void_p),
        ("hot_rows", c_void_p),
        ("n_hot", c_int32),
        ("hot_copies", c_int32),
        ("hot_buf", c_void_p),
        ("flags", c_int32),
        ("packed", c_void_p),
        ("pos", c_void_p),
        ("fixed_scale", c_void_p),
        ("mkeys", c_void_p),
        ("mvals", c_void_p),
        ("mtile", c_int32),
        ("hot_base", c_void_p),
        ("mrr", c_int32),
        ("n_pairs", c_int32),
        ("pair_a", c_int32 * 2),
        ("pair_b", c_int32 * 2),
        ("pair_tab", c_void_p * 2),
        ("mbase", c_void_p),
        ("l2_hot_bytes", ctypes.c_uint32 * ALTO_MAX_ORDER),
    ]


class CPullArgs(Structure):
    """alto_pull_args (include/alto_b200.h): K8/K9 slice buffers + pull."""
    _fields_ = [
        ("lay", POINTER(CLayout)),
        ("mkeys", c_void_p),
        ("mvals", c_void_p),
        ("value_dtype", c_int32),
        ("tile", c_int32),
        ("m", c_int64),
        ("mode", c_int32),
        ("rank", c_int32),
        ("factor_dtype", c_int32),
        ("out_dtype", c_int32),
        ("atomic", c_int32),
        ("pad_", c_int32),
        ("factors", c_void_p * ALTO_MAX_ORDER),
        ("out", c_void_p),
        ("slice_rec", c_void_p),
        ("rec", c_void_p),
        ("n_seg", c_int64),
        ("seg_row", c_void_p),
        ("n_chunks", c_int64),
        ("chunk_off", c_void_p),
        ("chunk_seg", c_void_p),
        ("seg_chunk_off", c_void_p),
        ("n_mseg", c_int64),
        ("mseg", c_void_p),
        ("part", c_void_p),
        ("slice_rows", c_void_p),
        ("mbase", c_void_p),
        ("n_pairs", c_int32),
        ("pair_a", c_int32 * 2),
        ("pair_b", c_int32 * 2),
        ("pair_tab", c_void_p * 2),
    ]


# (name, restype, argtypes) for every symbol of include/alto_b200.h
SIGNATURES = [
    ("alto_last_error", c_char_p, []),
    ("alto_version", c_int32, []),
    ("alto_tables_bytes", c_size_t, [POINTER(CLayout)]),
    ("alto_build_tables", c_int32, [POINTER(CLayout), c_void_p, c_void_p]),
    ("alto_linearize", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("alto_delinearize", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_sort_workspace_bytes", c_size_t, [c_int64, c_int32, c_int32]),
    ("alto_sort_pairs", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_size_t,
                                  c_void_p]),
    ("alto_find_duplicate", c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_partition", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                                 c_void_p]),
    ("alto_apply_flags", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int64, c_int32, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("alto_read_flags", c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    ("alto_clear_flags", c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    ("alto_mttkrp_ntiles", c_int64, [c_int64, c_int32]),
    ("alto_tile_intervals", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                      c_void_p]),
    ("alto_mttkrp", c_int32, [POINTER(CMttkrpArgs), c_void_p]),
    ("alto_pack_keys", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    ("alto_subtile_order", c_int32, [POINTER(CLayout), c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_mode_stream_workspace_bytes", c_size_t, [c_int64]),
    ("alto_coalesce_workspace_bytes", c_size_t, [c_int64, c_int32]),
    ("alto_coalesce", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_size_t, c_void_p]),
    ("alto_cpd_update", c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    ("alto_hot_copies", c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p,
                                  c_void_p, c_void_p]),
    ("alto_mode_stream", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int32,
                                   c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                   c_void_p]),
    ("alto_mstream_block", c_int32, [c_int32, c_int32, c_int32, c_int32, POINTER(c_int32), POINTER(c_int32)]),
    ("alto_topk_rows_workspace_bytes", c_size_t, [c_int64]),
    ("alto_hot_rows", c_int32, [c_void_p, c_int64, c_int32, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_size_t, c_void_p]),
    ("alto_hot_plan", c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("alto_row_counts", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_row_index_workspace_bytes", c_size_t, [c_int64, c_int64]),
    ("alto_row_index", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                 c_void_p, c_size_t, c_void_p]),
    ("alto_coord_max", c_int32, [POINTER(CLayout), c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    ("alto_mttkrp_pull", c_int32, [POINTER(CPullArgs), c_void_p]),
    ("alto_pull_slice_rows", c_int32, [POINTER(CLayout), c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p,
                                       c_void_p]),
    ("alto_mttkrp_exact", c_int32, [POINTER(CMttkrpArgs), c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    ("alto_mttkrp_coo", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, POINTER(c_void_p),
                                  c_void_p, c_int64, c_void_p]),
    ("alto_mttkrp_coo_workspace_bytes", c_size_t, [c_int64, c_int64]),
    ("alto_mttkrp_coo_ordered", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, POINTER(c_void_p),
                                          c_void_p, c_int64, c_void_p, c_size_t, c_void_p]),
    ("alto_cpd_workspace_bytes", c_size_t, [c_int32]),
    ("alto_gram", c_int32, [c_void_p, c_int32, c_int64, c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_hadamard_grams", c_int32, [POINTER(c_void_p), c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    ("alto_solve_normalize", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_fit_terms", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                 c_size_t, c_void_p]),
    ("alto_sumsq", c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_cast_f64_f32", c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    ("alto_cast_f32_f64", c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    ("alto_krp_pair", c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    ("alto_sumabs", c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_absmax", c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_fixed_scale", c_int32, [c_void_p, c_int32, c_void_p, c_void_p]),
    ("alto_fixed_to_float", c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p]),
    ("alto_pack_rows", c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_unpack_rows", c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_add_rows", c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    ("alto_gram_masked", c_int32, [c_void_p, c_int32, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_size_t,
                                   c_void_p]),
    ("alto_solve_rows", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_size_t,
                                  c_void_p]),
    ("alto_colsumsq", c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("alto_normalize", c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("alto_fit_inner_masked", c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                        c_void_p, c_size_t, c_void_p]),
]

_lib = None


def load(path: str | None = None):
    """Load the library (once) and bind every C ABI symbol."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"libalto_b200.so not found at {p}; build it with `make` or __graft_entry__.build()"
        )
    lib = ctypes.CDLL(p)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


class AltoDeviceError(RuntimeError):
    pass


def check(status: int, what: str = "") -> None:
    """Map a C ABI status to the reference's exception types."""
    if status == ALTO_OK:
        return
    msg = load().alto_last_error().decode(errors="replace")
    if status == ALTO_EINVAL:
        raise ValueError(msg)
    if status == ALTO_ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    raise AltoDeviceError(f"{what}: status {status}: {msg}")


def cuda_device():
    """The CUDA device the product path runs on; raises if there is none."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2102_10245_b200 needs a CUDA (B200) device; no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()
