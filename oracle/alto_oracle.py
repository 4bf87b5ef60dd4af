"""CPU oracle for the ALTO hot path — TEST INFRASTRUCTURE ONLY.

A NumPy/SciPy restatement of the reference algorithms (arXiv 2102.10245,
package `altotensor` at /root/reference/pkg/src/altotensor), one function per
reference function, each citing the file:line it follows.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; the product package (paper_2102_10245_b200) never does.

Parity pin: tests/test_oracle_golden.py checks every function here against
fixtures produced by running the reference itself in this container
(tests/golden/make_golden.py -> tests/golden/*.npz), including the
reference's own golden vectors (worked example of pkg/tests/conftest.py:8-20,
masks/positions of pkg/tests/test_layout.py:29-50, partitions/overlaps/flags
of pkg/tests/test_format.py:57-156).

Third-party arithmetic used by the reference and restated here: NumPy
(>=1.24; 2.3.5 installed) np.lexsort / np.add.at / np.unique, SciPy (>=1.10;
1.18.1 installed) cho_factor / cho_solve.
"""

from __future__ import annotations

import threading
from collections import namedtuple
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg

Layout = namedtuple("Layout", "dims bits positions masks total_bits width n_words")

U1 = np.uint64(1)


# --- layout.py ------------------------------------------------------------------

def build_layout(dims) -> Layout:
    """layout.py:31-35 (bits) and :74-102 (group interleave, width choice)."""
    dims = tuple(int(d) for d in dims)
    bits = tuple((d - 1).bit_length() for d in dims)
    total = sum(bits)
    if total > 128:
        raise ValueError("width overflow")
    width = 64 if total <= 64 else 128
    pos = [[] for _ in dims]
    nxt = 0
    for g in range(max(bits) if bits else 0):
        members = sorted((dims[n], n) for n in range(len(dims)) if bits[n] > g)
        for _, n in members:
            pos[n].append(nxt)
            nxt += 1
    masks = tuple(sum(1 << p for p in ps) for ps in pos)
    return Layout(dims, bits, tuple(map(tuple, pos)), masks, total, width, width // 64)


def encode(lay: Layout, coords) -> np.ndarray:
    """linearize_array, layout.py:148-160 (one pass per key bit)."""
    c = np.ascontiguousarray(coords, dtype=np.int64)
    out = np.zeros((c.shape[0], lay.n_words), dtype=np.uint64)
    for n, ps in enumerate(lay.positions):
        col = c[:, n].astype(np.uint64)
        for g, p in enumerate(ps):
            out[:, p >> 6] |= ((col >> np.uint64(g)) & U1) << np.uint64(p & 63)
    return out


def decode(lay: Layout, words, mode: int | None = None) -> np.ndarray:
    """extract_mode_array / delinearize_array, layout.py:163-182."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    modes = range(len(lay.dims)) if mode is None else [mode]
    cols = []
    for n in modes:
        acc = np.zeros(w.shape[0], dtype=np.uint64)
        for g, p in enumerate(lay.positions[n]):
            acc |= ((w[:, p >> 6] >> np.uint64(p & 63)) & U1) << np.uint64(g)
        cols.append(acc.astype(np.int64))
    return cols[0] if mode is not None else np.stack(cols, axis=1) if cols else np.zeros((w.shape[0], 0), np.int64)


# --- format.py ------------------------------------------------------------------

def sort_perm(words) -> np.ndarray:
    """_sort_by_words, format.py:79-82: lexsort with the last word primary."""
    return np.lexsort(tuple(words[:, k] for k in range(words.shape[1])))


def build(lay: Layout, coords, values):
    """build_alto, format.py:85-100 (encode, sort, co-permute, reject duplicates)."""
    words = encode(lay, coords)
    perm = sort_perm(words)
    words = words[perm]
    vals = np.asarray(values, dtype=np.float64)[perm]
    if words.shape[0] > 1 and (words[1:] == words[:-1]).all(axis=1).any():
        raise ValueError("duplicate coordinates; coalesce the tensor first")
    return words, vals


def offsets_for(m: int, count: int) -> np.ndarray:
    """format.py:136-140: sizes differ by <= 1, larger first."""
    base, extra = divmod(m, count)
    sizes = [base + 1] * extra + [base] * (count - extra)
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def as_int(row) -> int:
    return sum(int(x) << (64 * k) for k, x in enumerate(row))


def partition(lay: Layout, words, count: int):
    """partition, format.py:127-154 -> (offsets, intervals, spans)."""
    m = words.shape[0]
    if not 1 <= count <= max(m, 1):
        raise ValueError("partition count out of range")
    offs = offsets_for(m, count)
    coords = decode(lay, words)
    iv = np.empty((count, len(lay.dims), 2), dtype=np.int64)
    spans = []
    for l in range(count):
        a, b = offs[l], offs[l + 1]
        if a == b:
            iv[l, :, 0], iv[l, :, 1] = 0, -1
            continue
        iv[l, :, 0] = coords[a:b].min(axis=0)
        iv[l, :, 1] = coords[a:b].max(axis=0)
        spans.append((as_int(words[a]), as_int(words[b - 1])))
    return offs, iv, tuple(spans)


def merge_ranges(ranges):
    """_merge_ranges, format.py:199-207."""
    out = []
    for lo, hi in sorted(ranges):
        if out and lo <= out[-1][1] + 1:
            out[-1] = (out[-1][0], max(out[-1][1], hi))
        else:
            out.append((lo, hi))
    return tuple(out)


def plan(lay: Layout, nnz: int, intervals, mode: int, force: str | None = None, threshold: float = 4.0):
    """plan_conflicts, format.py:210-254 (literal pairwise overlap scan)."""
    reuse = nnz / lay.dims[mode]
    strategy = force or ("buffered" if reuse > threshold else "atomic")
    overlaps, flag_bit = None, None
    if strategy == "atomic":
        flag_bit = lay.total_bits if lay.total_bits < lay.width else None
        iv = [tuple(int(v) for v in intervals[l, mode]) for l in range(intervals.shape[0])]
        per = []
        for l, (lo, hi) in enumerate(iv):
            shared = []
            for j, (lo2, hi2) in enumerate(iv):
                a, b = max(lo, lo2), min(hi, hi2)
                if j != l and a <= b:
                    shared.append((a, b))
            per.append(merge_ranges(shared))
        overlaps = tuple(per)
    return {"strategy": strategy, "reuse": reuse, "overlaps": overlaps, "flag_bit": flag_bit}


def flag(lay: Layout, words, offsets, mode: int, overlaps, flag_bit: int) -> np.ndarray:
    """apply_boundary_flags, format.py:257-285."""
    out = words.copy()
    coords = decode(lay, words, mode)
    bit = np.uint64(1 << (flag_bit & 63))
    for l in range(len(offsets) - 1):
        a, b = offsets[l], offsets[l + 1]
        if a == b or not overlaps[l]:
            continue
        seg = coords[a:b]
        hit = np.zeros(b - a, dtype=bool)
        for lo, hi in overlaps[l]:
            hit |= (seg >= lo) & (seg <= hi)
        out[a + np.nonzero(hit)[0], flag_bit >> 6] |= bit
    return out


def read_flags(words, flag_bit: int) -> np.ndarray:
    """format.py:288-291."""
    return ((words[:, flag_bit >> 6] >> np.uint64(flag_bit & 63)) & U1).astype(bool)


# --- mttkrp.py ------------------------------------------------------------------

def mttkrp_coo(coords, values, factors, mode: int) -> np.ndarray:
    """mttkrp_oracle, mttkrp.py:64-77 (np.add.at in input order)."""
    rank = factors[0].shape[1]
    out = np.zeros((factors[mode].shape[0], rank))
    if len(values) == 0:
        return out
    prod = np.asarray(values, dtype=np.float64)[:, None].copy()
    for n in range(len(factors)):
        if n != mode:
            prod = prod * factors[n][coords[:, n]]
    np.add.at(out, coords[:, mode], prod)
    return out


def contributions(lay: Layout, words, values, factors, mode: int, a: int, b: int):
    """_contrib, mttkrp.py:80-105 for elements [a, b)."""
    c = decode(lay, words[a:b])
    prod = np.asarray(values[a:b], dtype=np.float64)[:, None]
    first = True
    for n in range(len(lay.dims)):
        if n == mode:
            continue
        g = factors[n][c[:, n]]
        prod = prod * g if first else prod * g
        first = False
    return c[:, mode], prod


CHUNK = 1 << 17  # mttkrp.py:39


def mttkrp_seq(lay: Layout, words, values, factors, mode: int) -> np.ndarray:
    """mttkrp_seq, mttkrp.py:108-117."""
    out = np.zeros((lay.dims[mode], factors[0].shape[1]))
    for a in range(0, words.shape[0], CHUNK):
        rows, prod = contributions(lay, words, values, factors, mode, a, min(a + CHUNK, words.shape[0]))
        np.add.at(out, rows, prod)
    return out


def _pool(workers: int, fn, n: int) -> None:
    """_run_workers, mttkrp.py:120-129."""
    ids = [w for w in range(workers) if w < n]
    if len(ids) <= 1:
        for w in ids:
            fn(w)
        return
    with ThreadPoolExecutor(max_workers=len(ids)) as ex:
        list(ex.map(fn, ids))


def mttkrp_buffered(lay, words, values, factors, mode, offsets, intervals, workers=1) -> np.ndarray:
    """_par_buffered, mttkrp.py:132-175 (stage into interval buffers, pull by row blocks)."""
    rank = factors[0].shape[1]
    dim = lay.dims[mode]
    count = len(offsets) - 1
    lo_v, hi_v = intervals[:, mode, 0], intervals[:, mode, 1]
    bufs = [None] * count

    def stage(w):
        for l in range(w, count, workers):
            buf = np.zeros((max(hi_v[l] - lo_v[l] + 1, 0), rank))
            for a in range(offsets[l], offsets[l + 1], CHUNK):
                rows, prod = contributions(lay, words, values, factors, mode, a, min(a + CHUNK, offsets[l + 1]))
                np.add.at(buf, rows - lo_v[l], prod)
            bufs[l] = buf

    _pool(workers, stage, count)
    out = np.zeros((dim, rank))
    cuts = [dim * w // workers for w in range(workers + 1)]

    def pull(w):
        r0, r1 = cuts[w], cuts[w + 1] - 1
        for l in range(count):
            a, b = max(int(lo_v[l]), r0), min(int(hi_v[l]), r1)
            if a <= b:
                out[a:b + 1] += bufs[l][a - lo_v[l]:b - lo_v[l] + 1]

    _pool(workers, pull, workers)
    return out


def mttkrp_atomic(lay, words, values, factors, mode, offsets, flag_bit, workers=1) -> np.ndarray:
    """_par_atomic, mttkrp.py:178-224 (plain adds for private rows, locked adds for flagged)."""
    rank = factors[0].shape[1]
    count = len(offsets) - 1
    flags = np.ones(words.shape[0], dtype=bool) if flag_bit is None else read_flags(words, flag_bit)
    out = np.zeros((lay.dims[mode], rank))
    lock = threading.Lock()

    def work(w):
        for l in range(w, count, workers):
            for a in range(offsets[l], offsets[l + 1], CHUNK):
                b = min(a + CHUNK, offsets[l + 1])
                rows, prod = contributions(lay, words, values, factors, mode, a, b)
                g = flags[a:b]
                if (~g).any():
                    np.add.at(out, rows[~g], prod[~g])
                if g.any():
                    uniq, inv = np.unique(rows[g], return_inverse=True)
                    packed = np.zeros((len(uniq), rank))
                    np.add.at(packed, inv, prod[g])
                    with lock:
                        out[uniq] += packed

    _pool(workers, work, count)
    return out


# --- cpd.py ---------------------------------------------------------------------

def gram(f) -> np.ndarray:
    """cpd.py:66-68."""
    return f.T @ f


def hadamard(factors, skip) -> np.ndarray:
    """_hadamard_grams, cpd.py:71-77."""
    r = factors[0].shape[1]
    v = np.ones((r, r))
    for n, f in enumerate(factors):
        if n != skip:
            v *= gram(f)
    return v


def solve(v, rhs) -> np.ndarray:
    """_solve_gram, cpd.py:80-95 (Cholesky, one ridge retry, else LinAlgError)."""
    errs = (np.linalg.LinAlgError, scipy.linalg.LinAlgError, ValueError)
    try:
        return scipy.linalg.cho_solve(scipy.linalg.cho_factor(v), rhs.T).T
    except errs:
        pass
    ridge = 1e-12 * np.trace(v) / v.shape[0]
    try:
        return scipy.linalg.cho_solve(scipy.linalg.cho_factor(v + ridge * np.eye(v.shape[0])), rhs.T).T
    except errs as exc:
        raise np.linalg.LinAlgError(f"singular even with ridge {ridge:g}: {exc}") from None


def update(factors, mode, m):
    """als_update, cpd.py:98-121 given the MTTKRP m."""
    new = solve(hadamard(factors, mode), m)
    w = np.linalg.norm(new, axis=0)
    return new / np.where(w == 0.0, 1.0, w), w


def fit_parts(norm_sq, factors, weights, m, mode) -> float:
    """fit_from_parts, cpd.py:124-138."""
    if norm_sq == 0.0:
        return 1.0
    model_sq = float(weights @ hadamard(factors, None) @ weights)
    inner = float(np.sum(m * factors[mode] * weights[None, :]))
    return 1.0 - np.sqrt(max(norm_sq - 2.0 * inner + model_sq, 0.0)) / np.sqrt(norm_sq)


def cpd_als(lay, words, values, rank, max_iters=50, tol=1e-5, seed=0, mttkrp_fn=None, init=None):
    """cpd_als, cpd.py:184-228 with the sequential MTTKRP (backend "seq").

    Returns (factors, weights, fit_history, iterations)."""
    rng = np.random.default_rng(seed)
    factors = init if init is not None else [rng.random((d, rank)) for d in lay.dims]
    factors = [np.asarray(f, dtype=np.float64) for f in factors]
    weights = np.ones(rank)
    values = np.asarray(values, dtype=np.float64)
    norm_sq = float(np.dot(values, values))
    run = mttkrp_fn or (lambda fs, n: mttkrp_seq(lay, words, values, fs, n))
    hist = [fit_parts(norm_sq, factors, weights, run(factors, 0), 0)]
    iters = 0
    for _ in range(max_iters):
        for n in range(len(lay.dims)):
            m = run(factors, n)
            factors[n], weights = update(factors, n, m)
        hist.append(fit_parts(norm_sq, factors, weights, m, len(lay.dims) - 1))
        iters += 1
        if abs(hist[-1] - hist[-2]) < tol:
            break
    return factors, weights, hist, iters


def rel_error(out, ref) -> float:
    """Relative Frobenius error (pkg/tests/conftest.py:35-38)."""
    d = float(np.linalg.norm(ref))
    e = float(np.linalg.norm(np.asarray(out) - ref))
    return e / d if d else e


def coalesce(coords, values):
    """COO coalesce (pkg/src/altotensor/coo.py:97-114): stable lexicographic
    row order with mode 0 primary, duplicates summed by np.bincount (i.e.
    sequentially in that order from 0.0).  -> (coords, values)."""
    c = np.ascontiguousarray(coords, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if c.shape[0] == 0:
        return c, v
    perm = np.lexsort(tuple(c[:, n] for n in range(c.shape[1] - 1, -1, -1)))
    c, v = c[perm], v[perm]
    new = np.ones(c.shape[0], dtype=bool)
    new[1:] = (c[1:] != c[:-1]).any(axis=1)
    return c[new], np.bincount(np.cumsum(new) - 1, weights=v)

