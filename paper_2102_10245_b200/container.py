"""`.alto` binary container <-> device-resident ALTO tensors.

Drop-in for pkg/src/altotensor/container.py (format :1-19, serialize :38-51,
deserialize :54-110, write_alto/read_alto :113-122): same little-endian
layout, same validation order and ContainerError messages, byte-identical
output.  The container's indices (M x width/8 bytes, least significant word
first) and float64 values are exactly the device layout of `AltoTensor.keys`
/ `.vals`, so reading a file is a chunked stream from disk through pinned
host buffers straight into HBM (no rebuild: no linearize, sort or duplicate
check), and writing streams the device arrays back out.  Float32 device
values are widened to the container's float64 on the device
(`alto_cast_f32_f64`, exact); `read_alto(..., dtype="float32")` narrows on
the device (`alto_cast_f64_f32`).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from . import _lib
from .format import AltoTensor
from .layout import build_masks

MAGIC = b"ALTO"
VERSION = 1
CHUNK_BYTES = 64 << 20  # staging chunk of the streamed file I/O


class ContainerError(ValueError):
    """Raised when a binary container is malformed or inconsistent (container.py:31-32)."""


def _torch():
    import torch

    return torch


def _header(tensor: AltoTensor) -> bytes:
    lay = tensor.layout
    wordlen = lay.width // 8
    out = bytearray(MAGIC)
    out += struct.pack("<BBBB", VERSION, lay.order, lay.width, 0)
    out += struct.pack(f"<{lay.order}Q", *lay.dims)
    out += struct.pack("<Q", tensor.nnz)
    for mask in lay.masks:
        out += int(mask).to_bytes(wordlen, "little")
    return bytes(out)


def _parse(head: bytes, total: int):
    """Validate the header against the total container length (container.py:56-101).
    -> (layout, nnz, offset of the indices)."""
    if total < 8 or len(head) < 8:
        raise ContainerError("truncated container (missing header)")
    if head[:4] != MAGIC:
        raise ContainerError(f"bad magic {head[:4]!r}, expected {MAGIC!r}")
    version, order, width, _reserved = struct.unpack_from("<BBBB", head, 4)
    if version != VERSION:
        raise ContainerError(f"unsupported container version {version}")
    if width not in (64, 128):
        raise ContainerError(f"unsupported index width {width}")
    if order < 1:
        raise ContainerError("container declares zero modes")
    off = 8
    if total < off + order * 8 + 8 or len(head) < off + order * 8 + 8:
        raise ContainerError("truncated container (missing dims)")
    dims = struct.unpack_from(f"<{order}Q", head, off)
    off += order * 8
    (nnz,) = struct.unpack_from("<Q", head, off)
    off += 8
    try:
        layout = build_masks(dims)
    except ValueError as exc:
        raise ContainerError(f"invalid dims {dims}: {exc}") from None
    if layout.width != width:
        raise ContainerError(f"declared width {width} does not match shape (needs {layout.width})")
    wordlen = width // 8
    expected = off + order * wordlen + nnz * wordlen + nnz * 8
    if total < expected:
        raise ContainerError(f"truncated container ({total} bytes, expected {expected})")
    if total > expected:
        raise ContainerError(f"trailing data ({total - expected} extra bytes)")
    for n in range(order):
        stored = int.from_bytes(head[off:off + wordlen], "little")
        if stored != layout.masks[n]:
            raise ContainerError(f"mask for mode {n} is {stored:#x}, layout derives {layout.masks[n]:#x}")
        off += wordlen
    return layout, nnz, off


def _head_len(order: int, width: int) -> int:
    return 8 + order * 8 + 8 + order * (width // 8)


def serialize(tensor: AltoTensor) -> bytes:
    """Encode an AltoTensor as container bytes (container.py:38-51)."""
    vals = tensor.values  # float64 host view (exact widening of float32 storage)
    return (_header(tensor) + np.ascontiguousarray(tensor.indices, dtype="<u8").tobytes()
            + np.ascontiguousarray(vals, dtype="<f8").tobytes())


def deserialize(data: bytes, dtype=None) -> AltoTensor:
    """Decode container bytes, verifying structure and masks (container.py:54-110);
    the tensor lands on the device (values float64, or float32 with dtype="float32")."""
    data = bytes(data)
    layout, nnz, off = _parse(data, len(data))
    nw = layout.n_words
    idx = np.frombuffer(data, dtype="<u8", count=nnz * nw, offset=off).reshape(nnz, nw)
    off += nnz * nw * 8
    vals = np.frombuffer(data, dtype="<f8", count=nnz, offset=off)
    t = AltoTensor(layout, idx.astype(np.uint64), vals.astype(np.float64))
    _check_coords(t)
    return _narrow(t, dtype)


def _check_coords(t: AltoTensor) -> None:
    """Every decoded coordinate must be below its mode extent: the masks
    admit values up to 2^b_n - 1, and a corrupt or crafted file must fail
    here (ContainerError) rather than drive out-of-range rows in a kernel."""
    if t.nnz == 0:
        return
    torch = _torch()
    from .layout import c_layout, device_tables

    lay = t.layout
    mx = torch.empty(lay.order, dtype=torch.int64, device=t.keys.device)
    _lib.check(_lib.load().alto_coord_max(c_layout(lay), device_tables(lay).data_ptr(), t.keys.data_ptr(), t.nnz,
                                          mx.data_ptr(), _lib.stream_ptr()), "alto_coord_max")
    for n, (c, d) in enumerate(zip(mx.cpu().tolist(), lay.dims)):
        if c >= d:
            raise ContainerError(f"coordinate {c} of mode {n} out of range for extent {d}")


def _narrow(t: AltoTensor, dtype) -> AltoTensor:
    if dtype is None or str(dtype) in ("float64", "torch.float64"):
        return t
    if str(dtype) not in ("float32", "torch.float32"):
        raise ValueError(f"dtype must be float32 or float64, got {dtype!r}")
    torch = _torch()
    v32 = torch.empty(t.nnz, dtype=torch.float32, device=t.vals.device)
    if t.nnz:
        _lib.check(_lib.load().alto_cast_f64_f32(t.vals.data_ptr(), v32.data_ptr(), t.nnz, _lib.stream_ptr()),
                   "alto_cast_f64_f32")
    return AltoTensor(t.layout, t.keys, v32)


def write_alto(tensor: AltoTensor, path: str) -> None:
    """Serialize `tensor` to a file (container.py:113-116), streaming the
    device arrays through a pinned staging buffer in CHUNK_BYTES pieces."""
    torch = _torch()
    lib = _lib.load()
    m = tensor.nnz
    nw = tensor.layout.n_words
    stage = torch.empty(CHUNK_BYTES, dtype=torch.uint8).pin_memory() if m else None
    with open(path, "wb") as f:
        f.write(_header(tensor))
        if not m:
            return
        keys = tensor.keys.view(-1)  # (m * nw,) int64, LS word first
        per = CHUNK_BYTES // 8
        for a in range(0, m * nw, per):
            b = min(m * nw, a + per)
            st = stage[:(b - a) * 8].view(torch.int64)
            st.copy_(keys[a:b])
            f.write(memoryview(stage[:(b - a) * 8].numpy()))
        vals = tensor.vals
        tmp = None
        if vals.dtype == torch.float32:
            tmp = torch.empty(min(m, per), dtype=torch.float64, device=vals.device)
        for a in range(0, m, per):
            b = min(m, a + per)
            st = stage[:(b - a) * 8].view(torch.float64)
            if tmp is not None:
                _lib.check(lib.alto_cast_f32_f64(vals[a:b].data_ptr(), tmp.data_ptr(), b - a, _lib.stream_ptr()),
                           "alto_cast_f32_f64")
                st.copy_(tmp[:b - a])
            else:
                st.copy_(vals[a:b])
            f.write(memoryview(stage[:(b - a) * 8].numpy()))


def read_alto(path: str, dtype=None) -> AltoTensor:
    """Read and verify a container file (container.py:119-122) straight into
    device memory: the header is validated against the file size first, then
    indices and values stream disk -> pinned buffer -> HBM in CHUNK_BYTES
    pieces (two staging buffers, so a disk read overlaps the previous copy)."""
    torch = _torch()
    total = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(min(total, 8))
        if len(head) == 8 and head[:4] == MAGIC and head[6] in (64, 128):
            head += f.read(_head_len(head[5], head[6]) - 8)
        layout, nnz, off = _parse(head, total)
        dev = _lib.cuda_device()
        nw = layout.n_words
        keys = torch.empty((nnz, nw), dtype=torch.int64, device=dev)
        vals = torch.empty(nnz, dtype=torch.float64, device=dev)
        if nnz:
            f.seek(off)
            stages = [torch.empty(CHUNK_BYTES, dtype=torch.uint8).pin_memory() for _ in range(2)]
            done = [None, None]
            stream = torch.cuda.current_stream(dev)

            def pump(dst_bytes):
                n = dst_bytes.numel()
                k = 0
                for a in range(0, n, CHUNK_BYTES):
                    b = min(n, a + CHUNK_BYTES)
                    s = k & 1
                    if done[s] is not None:
                        done[s].synchronize()  # staging buffer s is free again
                    view = stages[s][:b - a]
                    got = f.readinto(memoryview(view.numpy()))
                    if got != b - a:
                        raise ContainerError("truncated container (short read)")
                    dst_bytes[a:b].copy_(view, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    done[s] = ev
                    k += 1

            pump(keys.view(torch.uint8).view(-1))
            pump(vals.view(torch.uint8).view(-1))
            torch.cuda.current_stream(dev).synchronize()
    t = AltoTensor(layout, keys, vals)
    _check_coords(t)
    return _narrow(t, dtype)
