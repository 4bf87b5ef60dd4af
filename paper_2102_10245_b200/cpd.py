"""CP-ALS with the whole step on the B200: drop-in for pkg/src/altotensor/cpd.py.

Per mode: MTTKRP (device engine chosen by `backend`), Hadamard of Grams
(K10), Cholesky solve with ridge retry + column normalisation (K11/K12),
Gram refresh; per sweep: fit terms (K13).  Only the two fit scalars and a
status word cross to the host per sweep.  Factor init is the reference's
own NumPy draw (`default_rng(seed).random((I_n, R))`, cpd.py:206-210), so
runs start from identical factors.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .format import (AltoTensor, Strategy, apply_boundary_flags, partition,
                     plan_conflicts)
from .mttkrp import (F32_ACCUMULATE, _check_factors, factors_to_device, mttkrp_deterministic,
                     mttkrp_seq, mttkrp_stream)

BACKENDS = ("seq", "oracle", "auto", "buffered", "atomic")
# Replay the per-mode updates of a sweep as one CUDA graph (after the first sweep)
CPD_GRAPHS = True
# alto_cpd_update flags (ALTO_CPD_SCALAR = 1: scalar substitution instead of the rank-16 DMMA path)
CPD_UPDATE_FLAGS = 0


def _torch():
    import torch

    return torch


@dataclass
class CpModel:
    """Rank-R CP model: weights and unit-column factors (cpd.py:39-63)."""

    factors: list
    weights: np.ndarray
    fit_history: list = field(default_factory=list)
    iterations: int = 0

    @property
    def rank(self) -> int:
        return int(np.asarray(self.weights).shape[0])

    def to_dense(self) -> np.ndarray:
        """Dense reconstruction (small shapes only), computed on the device."""
        torch = _torch()
        dev = _lib.cuda_device()
        fs = [torch.as_tensor(np.asarray(f, dtype=np.float64), device=dev) for f in self.factors]
        w = torch.as_tensor(np.asarray(self.weights, dtype=np.float64), device=dev)
        dims = tuple(int(f.shape[0]) for f in fs)
        out = torch.zeros(dims, dtype=torch.float64, device=dev)
        for r in range(self.rank):
            term = w[r]
            for n, f in enumerate(fs):
                shape = [1] * len(dims)
                shape[n] = dims[n]
                term = term * f[:, r].reshape(shape)
            out += term
        return out.cpu().numpy()


class _Workspace:
    """Per-rank device scratch for the CP-ALS kernels."""

    def __init__(self, rank: int, dev):
        torch = _torch()
        lib = _lib.load()
        self.bytes = int(lib.alto_cpd_workspace_bytes(rank))
        self.buf = torch.empty(self.bytes, dtype=torch.uint8, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.terms = torch.zeros(2, dtype=torch.float64, device=dev)
        self.scalar = torch.zeros(1, dtype=torch.float64, device=dev)


def gram_device(f, ws: _Workspace, out=None):
    torch = _torch()
    rank = int(f.shape[1])
    if out is None:
        out = torch.empty((rank, rank), dtype=torch.float64, device=f.device)
    code = _lib.ALTO_F32 if f.dtype == torch.float32 else _lib.ALTO_F64
    _lib.check(_lib.load().alto_gram(f.data_ptr(), code, int(f.shape[0]), rank, out.data_ptr(), ws.buf.data_ptr(),
                                     ws.bytes, _lib.stream_ptr()), "alto_gram")
    return out


def hadamard_device(grams: list, skip: int | None, out=None):
    torch = _torch()
    rank = int(grams[0].shape[0])
    if out is None:
        out = torch.empty((rank, rank), dtype=torch.float64, device=grams[0].device)
    arr = (ctypes.c_void_p * len(grams))(*[g.data_ptr() for g in grams])
    _lib.check(_lib.load().alto_hadamard_grams(arr, len(grams), -1 if skip is None else int(skip), rank,
                                               out.data_ptr(), _lib.stream_ptr()), "alto_hadamard_grams")
    return out


def solve_device(v, m, ws: _Workspace, x64=None, x32=None, lam=None):
    """X V = M, lambda = column norms, X /= lambda; status left in ws.status."""
    torch = _torch()
    rows, rank = int(m.shape[0]), int(m.shape[1])
    if x64 is None:
        x64 = torch.empty((rows, rank), dtype=torch.float64, device=m.device)
    if lam is None:
        lam = torch.empty(rank, dtype=torch.float64, device=m.device)
    _lib.check(_lib.load().alto_solve_normalize(v.data_ptr(), m.data_ptr(), rows, rank, x64.data_ptr(),
                                                None if x32 is None else x32.data_ptr(), lam.data_ptr(),
                                                ws.status.data_ptr(), ws.buf.data_ptr(), ws.bytes,
                                                _lib.stream_ptr()), "alto_solve_normalize")
    return x64, lam


def fit_terms_device(m, f, lam, vall, ws: _Workspace):
    _lib.check(_lib.load().alto_fit_terms(m.data_ptr(), f.data_ptr(), lam.data_ptr(), vall.data_ptr(),
                                          int(m.shape[0]), int(m.shape[1]), ws.terms.data_ptr(), ws.buf.data_ptr(),
                                          ws.bytes, _lib.stream_ptr()), "alto_fit_terms")
    return ws.terms


def sumsq_device(vals, ws: _Workspace) -> float:
    torch = _torch()
    code = _lib.ALTO_F32 if vals.dtype == torch.float32 else _lib.ALTO_F64
    _lib.check(_lib.load().alto_sumsq(vals.data_ptr(), code, int(vals.shape[0]), ws.scalar.data_ptr(),
                                      ws.buf.data_ptr(), ws.bytes, _lib.stream_ptr()), "alto_sumsq")
    return float(ws.scalar.item())


def _raise_singular(v) -> None:
    v = v.cpu().numpy()
    ridge = 1e-12 * np.trace(v) / v.shape[0]
    raise np.linalg.LinAlgError(f"normal equations singular even with ridge {ridge:g}")


def gram(factor) -> np.ndarray:
    """F^T F in float64 (cpd.py:66-68), computed on device."""
    fd = factors_to_device([factor])[0]
    ws = _Workspace(int(fd.shape[1]), fd.device)
    g = gram_device(fd, ws)
    return g if isinstance(factor, _torch().Tensor) else g.cpu().numpy()


def fit_from_terms(norm_sq: float, inner: float, model_sq: float) -> float:
    """1 - ||X - X~|| / ||X|| from the fit terms (cpd.py:124-138)."""
    if norm_sq == 0.0:
        return 1.0
    resid = max(norm_sq - 2.0 * inner + model_sq, 0.0)
    return 1.0 - math.sqrt(resid) / math.sqrt(norm_sq)


def _device_fit(norm_sq, fdev64, grams, lam, m_dev, mode, ws) -> float:
    vall = hadamard_device(grams, None)
    t = fit_terms_device(m_dev, fdev64[mode], lam, vall, ws).cpu().numpy()
    return float(fit_from_terms(norm_sq, float(t[0]), float(t[1])))


def als_update(tensor: AltoTensor, model: CpModel, mode: int,
               mttkrp_fn: Callable[[Sequence[np.ndarray], int], np.ndarray] | None = None):
    """One least-squares factor update (cpd.py:98-121); model is not mutated."""
    torch = _torch()
    _check_factors(tensor.layout.dims, model.factors, mode)
    if mttkrp_fn is None:
        m = mttkrp_seq(tensor, model.factors, mode)
    else:
        m = mttkrp_fn(model.factors, mode)
    fdev = factors_to_device(model.factors, torch.float64)
    rank = int(fdev[0].shape[1])
    ws = _Workspace(rank, fdev[0].device)
    grams = [gram_device(f, ws) for f in fdev]
    v = hadamard_device(grams, mode)
    m_dev = factors_to_device([m], torch.float64)[0]
    x64, lam = solve_device(v, m_dev, ws)
    if int(ws.status.item()) == 2:
        _raise_singular(v)
    return x64.cpu().numpy(), lam.cpu().numpy(), (m if not isinstance(m, torch.Tensor) else m.cpu().numpy())


def fit(tensor: AltoTensor, model: CpModel, last_mttkrp, last_mode: int) -> float:
    """Model fit from one mode's MTTKRP (cpd.py:141-146)."""
    torch = _torch()
    fdev = factors_to_device(model.factors, torch.float64)
    ws = _Workspace(int(fdev[0].shape[1]), fdev[0].device)
    norm_sq = sumsq_device(tensor.vals, ws)
    grams = [gram_device(f, ws) for f in fdev]
    lam = torch.as_tensor(np.asarray(model.weights, dtype=np.float64), device=fdev[0].device)
    m_dev = factors_to_device([last_mttkrp], torch.float64)[0]
    return _device_fit(norm_sq, fdev, grams, lam, m_dev, last_mode, ws)


class DeviceBackend:
    """Binds an MTTKRP engine to a tensor, with per-mode plans built once
    (cpd.py:149-181).  run(fdev, mode) -> (I_mode, R) float64 device tensor."""

    def __init__(self, tensor: AltoTensor, backend: str, workers: int, partitions: int | None):
        if backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}, got {backend!r}")
        self.tensor = tensor
        self.backend = backend
        order = tensor.layout.order
        self.engine = ["exact"] * order
        self.offsets = [None] * order
        if backend in ("seq", "oracle"):
            # The reference's oracle backend delinearizes the ALTO tensor in
            # stored order and runs np.add.at in that order (cpd.py:159-162),
            # i.e. the same arithmetic order as mttkrp_seq: the exact-order
            # engine reproduces both (deterministically).
            return
        force = {"auto": None, "buffered": Strategy.BUFFERED, "atomic": Strategy.ATOMIC}[backend]
        count = max(min(partitions if partitions is not None else workers, tensor.nnz), 1)
        parts = partition(tensor, count)
        for mode in range(order):
            plan = plan_conflicts(tensor, parts, mode, force_strategy=force)
            if plan.strategy is Strategy.BUFFERED:
                self.engine[mode] = "exact"
                self.offsets[mode] = np.asarray(parts.offsets)
            else:
                if plan.flag_bit is not None:
                    apply_boundary_flags(tensor, plan)  # validated like the reference (cpd.py:172-176)
                # Atomic backend: the mode-stream kernel (per-row-run atomic
                # merges, Zipf-head rows through float64-summed replicated
                # copies) — the fastest float32 path; mttkrp_par with an
                # Atomic plan runs the pull engine's flag-exact atomic scheme
                self.engine[mode] = "stream"

    def run(self, fdev: list, mode: int, out=None, allow_f32: bool = False):
        """allow_f32: the streaming engine may return its float32 result (float32
        tensor and factors: identical to the float64 upcast the API returns)."""
        torch = _torch()
        eng = self.engine[mode]
        if eng == "stream":
            if (allow_f32 and out is None and F32_ACCUMULATE and self.tensor.vals.dtype == torch.float32
                    and fdev[0].dtype == torch.float32):
                return mttkrp_stream(self.tensor, fdev, mode, out_dtype=torch.float32)
            return mttkrp_stream(self.tensor, fdev, mode, out=out)
        if eng == "coo":
            return _coo_run(self.tensor, fdev, mode)
        od = None
        if (allow_f32 and out is None and self.tensor.vals.dtype == torch.float32
                and fdev[0].dtype == torch.float32):
            od = torch.float32  # the pull engine may hand its float32 rows straight to the update
        return mttkrp_deterministic(self.tensor, fdev, mode, self.offsets[mode], out=out, out_dtype=od)


def _coo_run(tensor: AltoTensor, fdev: list, mode: int):
    """COO-oracle backend on device: decode once, then the COO kernel."""
    torch = _torch()
    from .layout import delinearize_device

    coords = tensor._cache.get("coo_coords")
    if coords is None:
        coords = delinearize_device(tensor.layout, tensor.keys, -1)
        tensor._cache["coo_coords"] = coords
    rank = int(fdev[0].shape[1])
    out = torch.empty((tensor.layout.dims[mode], rank), dtype=torch.float64, device=coords.device)
    vals = tensor.vals.double()
    f64 = [f.double() for f in fdev]
    arr = (ctypes.c_void_p * len(f64))(*[f.data_ptr() for f in f64])
    _lib.check(_lib.load().alto_mttkrp_coo(coords.data_ptr(), vals.data_ptr(), tensor.nnz, tensor.layout.order,
                                           mode, rank, arr, out.data_ptr(), tensor.layout.dims[mode],
                                           _lib.stream_ptr()), "alto_mttkrp_coo")
    return out


class DeviceCpAls:
    """Device-resident CP-ALS state: float64 master factors, optional float32
    gather copies (for float32 tensors), cached Grams."""

    def __init__(self, tensor: AltoTensor, rank: int, seed: int, backend: str = "seq", workers: int = 1,
                 partitions: int | None = None, init_factors=None):
        torch = _torch()
        self.tensor = tensor
        self.rank = rank
        dims = tensor.layout.dims
        if init_factors is None:
            rng = np.random.default_rng(seed)
            init_factors = [rng.random((d, rank)) for d in dims]
        self.f64 = factors_to_device(init_factors, torch.float64)
        dev = self.f64[0].device
        self.use32 = tensor.vals.dtype == torch.float32
        self.f32 = [f.float() for f in self.f64] if self.use32 else None
        self.ws = _Workspace(rank, dev)
        self.backend = DeviceBackend(tensor, backend, workers, partitions)
        self.grams = [gram_device(f, self.ws) for f in self.f64]
        self.lam = torch.ones(rank, dtype=torch.float64, device=dev)
        self.norm_sq = sumsq_device(tensor.vals, self.ws)
        self.v = torch.empty((rank, rank), dtype=torch.float64, device=dev)
        self.m_last = None
        self._graph = None
        self._graph_m = None

    def gather_factors(self):
        return self.f32 if self.use32 else self.f64

    def mttkrp(self, mode: int):
        return self.backend.run(self.gather_factors(), mode)

    def update(self, mode: int):
        """One factor update on device; no host sync.  Ranks 16/32 use the
        fused update (alto_cpd_update: solve, norms, normalise, Gram in two
        streaming passes, reading a float32 MTTKRP directly); other ranks the
        separate K11/K12/K10 kernels."""
        torch = _torch()
        fused = self.rank in (16, 32)
        m = self.backend.run(self.gather_factors(), mode, allow_f32=fused)
        hadamard_device(self.grams, mode, out=self.v)
        if fused:
            code = _lib.ALTO_F32 if m.dtype == torch.float32 else _lib.ALTO_F64
            x32 = self.f32[mode] if self.use32 else None
            _lib.check(_lib.load().alto_cpd_update(
                self.v.data_ptr(), m.data_ptr(), code, int(m.shape[0]), self.rank, self.f64[mode].data_ptr(),
                None if x32 is None else x32.data_ptr(), self.lam.data_ptr(), self.grams[mode].data_ptr(),
                self.ws.status.data_ptr(), CPD_UPDATE_FLAGS, self.ws.buf.data_ptr(), self.ws.bytes,
                _lib.stream_ptr()), "alto_cpd_update")
        else:
            solve_device(self.v, m, self.ws, x64=self.f64[mode], x32=self.f32[mode] if self.use32 else None,
                         lam=self.lam)
            gram_device(self.f64[mode], self.ws, out=self.grams[mode])
        self.m_last = m
        return m

    def check_status(self) -> None:
        if int(self.ws.status.item()) == 2:
            _raise_singular(self.v)

    def fit(self, m, mode: int) -> float:
        torch = _torch()
        if m.dtype == torch.float32:
            m64 = torch.empty(m.shape, dtype=torch.float64, device=m.device)
            _lib.check(_lib.load().alto_cast_f32_f64(m.data_ptr(), m64.data_ptr(), m.numel(), _lib.stream_ptr()),
                       "alto_cast_f32_f64")
            m = m64
        return _device_fit(self.norm_sq, self.f64, self.grams, self.lam, m, mode, self.ws)

    def _updates(self):
        m = None
        for mode in range(self.tensor.layout.order):
            m = self.update(mode)
        return m

    def sweep(self) -> float:
        """One ALS sweep (all modes) and its fit.  After the first (eager)
        sweep the per-mode updates are captured once in a CUDA graph and
        replayed: every kernel and workspace is static by then (plans,
        hot-row copies and launch configurations are cached), and a replay
        removes the host launch gaps between the ~30 small launches of a
        sweep.  Set CPD_GRAPHS = False to run eagerly."""
        torch = _torch()
        order = self.tensor.layout.order
        if not CPD_GRAPHS or self._graph is False:
            m = self._updates()
        elif self._graph is None:
            m = self._updates()  # eager warm-up: builds every cache the capture needs
            torch.cuda.synchronize()
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._graph_m = self._updates()
                self._graph = g
                self.m_last = m  # the capture recorded, but did not run, the updates
            except Exception:  # capture unsupported here: stay eager (same kernels)
                self._graph = False
                torch.cuda.synchronize()
        else:
            self._graph.replay()
            m = self._graph_m
            self.m_last = m
        self.check_status()
        return self.fit(m, order - 1)


def cpd_als(tensor: AltoTensor, rank: int, max_iters: int = 50, tol: float = 1e-5, seed: int = 0,
            backend: str = "seq", workers: int = 1, partitions: int | None = None) -> CpModel:
    """Rank-`rank` CP-ALS (cpd.py:184-228) with every step on the device."""
    if rank < 1:
        raise ValueError("rank must be at least 1")
    if max_iters < 0:
        raise ValueError("max_iters must be nonnegative")
    if backend not in BACKENDS:
        raise ValueError(f"backend must be one of {BACKENDS}, got {backend!r}")
    st = DeviceCpAls(tensor, rank, seed, backend, workers, partitions)
    m0 = st.mttkrp(0)
    history = [st.fit(m0, 0)]
    iters = 0
    for _ in range(max_iters):
        history.append(st.sweep())
        iters += 1
        if abs(history[-1] - history[-2]) < tol:
            break
    model = CpModel(factors=[f.cpu().numpy() for f in st.f64], weights=st.lam.cpu().numpy(),
                    fit_history=history, iterations=iters)
    return model


def save_factors_csv(model: "CpModel", out_dir: str, prefix: str = "factor") -> list:
    """One CSV per factor matrix, `<prefix>_<mode>.csv` with one-based mode
    numbers, a row per index (cpd.py:231-242); returns the paths written.
    Host I/O, not on the device path."""
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for n, fac in enumerate(model.factors, start=1):
        path = os.path.join(out_dir, f"{prefix}_{n}.csv")
        np.savetxt(path, np.asarray(fac), delimiter=",")
        paths.append(path)
    return paths
