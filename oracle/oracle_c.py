"""ctypes binding of the C oracle (oracle/mttkrp_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Used by tests/ (full-size parity at BASELINE.json's sizes) and never by the
product package.  Restates /root/reference/pkg/src/altotensor/mttkrp.py:64-77
(mttkrp_oracle) bitwise; see the C file's header.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liboracle_c.so")
_LIB = None


def load():
    """Load (building if needed: gcc is on the build container and the box) the C oracle."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
        lib = ctypes.CDLL(LIB_PATH)
        lib.oracle_mttkrp_coo.restype = ctypes.c_int
        lib.oracle_mttkrp_coo.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        lib.oracle_diff_norms.restype = None
        lib.oracle_diff_norms.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
        _LIB = lib
    return _LIB


def host_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def mttkrp_coo(coords, values, factors, mode: int, threads: int | None = None) -> np.ndarray:
    """fp64 MTTKRP over a coordinate list, bitwise equal to the reference's
    mttkrp_oracle.  `coords`: (M, N) integer array or a list of N per-mode
    int32 arrays; `values`: float32 or float64 (M,); `factors`: float64 (I_n, R)."""
    lib = load()
    if isinstance(coords, np.ndarray):
        cols = [np.ascontiguousarray(coords[:, n], dtype=np.int32) for n in range(coords.shape[1])]
    else:
        cols = [np.ascontiguousarray(c, dtype=np.int32) for c in coords]
    order = len(cols)
    m = cols[0].shape[0] if order else 0
    vals = np.ascontiguousarray(values)
    if vals.dtype not in (np.float32, np.float64):
        vals = vals.astype(np.float64)
    fac = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    rank = fac[0].shape[1]
    dim = fac[mode].shape[0]
    out = np.empty((dim, rank), dtype=np.float64)
    cptr = (ctypes.c_void_p * order)(*[c.ctypes.data for c in cols])
    fptr = (ctypes.c_void_p * order)(*[f.ctypes.data for f in fac])
    rc = lib.oracle_mttkrp_coo(order, mode, m, rank, cptr, vals.ctypes.data, 1 if vals.dtype == np.float32 else 0,
                               fptr, out.ctypes.data, dim, threads or host_threads())
    if rc != 0:
        raise ValueError(f"oracle_mttkrp_coo failed ({rc})")
    return out


def rel_error(got, ref: np.ndarray, threads: int | None = None) -> float:
    """||got - ref||_F / ||ref||_F (pkg/tests/conftest.py:35-38) in float64;
    `got` float32 or float64, same shape as `ref`."""
    lib = load()
    a = np.ascontiguousarray(got)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    b = np.ascontiguousarray(ref, dtype=np.float64)
    assert a.size == b.size
    d2, n2 = ctypes.c_double(), ctypes.c_double()
    lib.oracle_diff_norms(a.ctypes.data, 1 if a.dtype == np.float32 else 0, b.ctypes.data, b.size,
                          threads or host_threads(), ctypes.byref(d2), ctypes.byref(n2))
    if n2.value == 0.0:
        return float(np.sqrt(d2.value))
    return float(np.sqrt(d2.value / n2.value))
