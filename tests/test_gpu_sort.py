"""K2 radix sort and K3 duplicate detection through the C ABI, against
NumPy (stable argsort / lexsort) — bit-exact, including stability."""

import numpy as np
import pytest

from paper_2102_10245_b200 import _lib

pytestmark = pytest.mark.gpu


def run_sort(keys_u64, payload, total_bits):
    import torch

    lib = _lib.load()
    m, w = keys_u64.shape
    k = torch.from_numpy(keys_u64.view(np.int64).copy()).cuda()
    p = None if payload is None else torch.from_numpy(payload.copy()).cuda()
    pb = 0 if payload is None else payload.dtype.itemsize
    ws_bytes = lib.alto_sort_workspace_bytes(m, w, pb)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device="cuda")
    _lib.check(lib.alto_sort_pairs(k.data_ptr(), None if p is None else p.data_ptr(), m, w, pb, total_bits,
                                   ws.data_ptr(), ws_bytes, _lib.stream_ptr()))
    return k.cpu().numpy().view(np.uint64), None if p is None else p.cpu().numpy()


@pytest.mark.parametrize("m", [1, 2, 31, 4095, 4096, 4097, 100_000, 1_000_003])
@pytest.mark.parametrize("w,bits", [(1, 53), (1, 8), (1, 64), (2, 71), (2, 128)])
def test_sort_matches_numpy_stable(m, w, bits):
    rng = np.random.default_rng(m + bits)
    keys = np.zeros((m, w), dtype=np.uint64)
    for j in range(w):
        nb = min(64, bits - 64 * j)
        if nb <= 0:
            continue
        hi = (1 << nb) - 1
        keys[:, j] = rng.integers(0, hi, size=m, dtype=np.uint64, endpoint=True)
    keys[: m // 3] = keys[m // 3: 2 * (m // 3)]  # force ties so stability is observable
    payload = np.arange(m, dtype=np.uint32)
    out_k, out_p = run_sort(keys, payload, bits)
    perm = np.lexsort(tuple(keys[:, j] for j in range(w)))  # stable, last word primary
    assert np.array_equal(out_k, keys[perm])
    assert np.array_equal(out_p, payload[perm])


def test_sort_payload_sizes():
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 1 << 40, size=(50_000, 1), dtype=np.uint64)
    perm = np.argsort(keys[:, 0], kind="stable")
    for pay in (None, rng.random(50_000), rng.random(50_000).astype(np.float32)):
        k, p = run_sort(keys, pay, 40)
        assert np.array_equal(k[:, 0], keys[perm, 0])
        if pay is not None:
            assert np.array_equal(p, pay[perm])


def test_find_duplicate():
    import torch

    lib = _lib.load()
    for w in (1, 2):
        keys = np.arange(10 * w, dtype=np.uint64).reshape(10, w)
        keys[7] = keys[6]
        k = torch.from_numpy(keys.view(np.int64)).cuda()
        first = torch.empty(1, dtype=torch.int64, device="cuda")
        _lib.check(lib.alto_find_duplicate(k.data_ptr(), 10, w, first.data_ptr(), _lib.stream_ptr()))
        assert int(first.item()) == 7
        keys[7, 0] += np.uint64(100)
        k = torch.from_numpy(keys.view(np.int64)).cuda()
        _lib.check(lib.alto_find_duplicate(k.data_ptr(), 10, w, first.data_ptr(), _lib.stream_ptr()))
        assert int(first.item()) == -1
