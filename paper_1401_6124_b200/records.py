"""Signature files written straight from GPU signature blocks.

The reference writes records one object at a time in Python
(``write_signatures_text`` / ``write_signatures_binary``, minhash.py:140-206;
``cli._cmd_sign``, cli.py:205-230).  Here a CSR batch is signed chunk by chunk on
the device, each chunk's records are formatted by libmhb kernels into the exact
bytes the reference writes, and the bytes stream to the file.  The files read
back with ``read_signatures_text`` / ``read_signatures_binary`` (and with the
reference's own readers).
"""
from __future__ import annotations

import threading

import numpy as np

from . import _lib
from .families import Family
from .minhash import signatures_csr


def _dtype_code(sig):
    import torch

    return _lib.OUT_I64 if sig.dtype == torch.int64 else _lib.OUT_U32


def format_binary(sig, obj_ids=None, first_id: int = 0):
    """uint64 device tensor [S*(N+2)]: per record (id, N, ids...) as the reference's
    little-endian binary record (minhash.py:182-188)."""
    import torch

    lib = _lib.load()
    s, n = sig.shape
    out = torch.empty(s * (n + 2), dtype=torch.uint64, device=sig.device)
    oid = None
    if obj_ids is not None:
        oid = torch.as_tensor(obj_ids, dtype=torch.int64, device=sig.device).contiguous()
    with torch.cuda.device(sig.device):
        rc = lib.mhb_format_binary_records(sig.contiguous().data_ptr(), _dtype_code(sig), s, n,
                                           oid.data_ptr() if oid is not None else None, int(first_id),
                                           out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    return out


def format_text(sig, obj_ids=None, first_id: int = 0):
    """uint8 device tensor: the lines "id N x0 ... xN-1\\n" of every record, byte for byte
    what write_signatures_text writes (minhash.py:154-161)."""
    import torch

    lib = _lib.load()
    s, n = sig.shape
    sig = sig.contiguous()
    oid = None
    if obj_ids is not None:
        oid = torch.as_tensor(obj_ids, dtype=torch.int64, device=sig.device).contiguous()
    lens = torch.empty(s, dtype=torch.int64, device=sig.device)
    with torch.cuda.device(sig.device):
        stream = torch.cuda.current_stream().cuda_stream
        _lib.check(lib.mhb_text_record_lengths(sig.data_ptr(), _dtype_code(sig), s, n,
                                               oid.data_ptr() if oid is not None else None, int(first_id),
                                               lens.data_ptr(), stream))
        offsets = torch.zeros(s, dtype=torch.int64, device=sig.device)
        if s > 1:
            torch.cumsum(lens[:-1], 0, out=offsets[1:])
        total = int(offsets[-1] + lens[-1]) if s else 0
        out = torch.empty(total, dtype=torch.uint8, device=sig.device)
        _lib.check(lib.mhb_format_text_records(sig.data_ptr(), _dtype_code(sig), s, n,
                                               oid.data_ptr() if oid is not None else None, int(first_id),
                                               offsets.data_ptr(), out.data_ptr(), stream))
    return out


_PINNED = threading.local()  # per thread: slot -> pinned uint8 host buffer, reused across calls


def _pinned(slot: int, nbytes: int):
    import torch

    bufs = getattr(_PINNED, "bufs", None)
    if bufs is None:
        bufs = _PINNED.bufs = {}
    buf = bufs.get(slot)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        bufs[slot] = buf
    return buf[:nbytes]


def write_signatures_csr(path, indptr, ids, family: Family, fmt: str = "binary", obj_ids=None,
                         first_id: int = 0, chunk_bytes: int = 64 << 20) -> int:
    """Sign every set of a CSR batch and write the records to `path`.

    fmt: "binary" (LE u64 records) or "text" ("id N ids..." lines).  obj_ids: one id per
    set (default first_id + row).  Works on device tensors or numpy arrays.  The batch
    is processed in chunks of about `chunk_bytes` of formatted output; each chunk's
    bytes land in one of two pinned host buffers while the previous chunk is written
    to the file.  Returns the number of records written."""
    import torch

    if fmt not in ("binary", "text"):
        raise ValueError(f"fmt must be 'binary' or 'text', got {fmt!r}")
    dev = torch.device("cuda", torch.cuda.current_device())
    ip = torch.as_tensor(np.asarray(indptr) if not torch.is_tensor(indptr) else indptr, dtype=torch.int64)
    x = ids if torch.is_tensor(ids) else torch.from_numpy(np.asarray(ids))
    n_sets = ip.numel() - 1
    oids = None if obj_ids is None else np.asarray(obj_ids, dtype=np.int64)
    per_record = (family.size + 2) * 8 if fmt == "binary" else family.size * 11 + 24
    step = max(1, chunk_bytes // per_record)
    ip_h = ip.cpu().numpy()
    written = 0
    pending = None  # (pinned host view, event) of the chunk in flight
    slot = 0
    with open(path, "wb") as fh:
        fd, pos = fh.fileno(), 0

        def flush(view):  # concurrent pwrite of the chunk (page-cache copies in parallel)
            nonlocal pos
            _pwrite_parallel(fd, memoryview(view.numpy()), pos)
            pos += view.numel()

        for s0 in range(0, n_sets, step):
            s1 = min(n_sets, s0 + step)
            lo, hi = int(ip_h[s0]), int(ip_h[s1])
            cip = torch.as_tensor(ip_h[s0:s1 + 1] - lo).to(dev, non_blocking=True)
            cx = x[lo:hi]
            if cx.dtype != torch.uint32:
                cx = cx.to(torch.int64).to(torch.uint32) if cx.dtype != torch.int64 else cx.to(torch.uint32)
            cx = cx.to(dev, non_blocking=True)
            sig = signatures_csr(cip, cx, family, out_dtype="uint32")
            chunk_ids = None if oids is None else oids[s0:s1]
            buf = format_binary(sig, chunk_ids, first_id + s0) if fmt == "binary" else \
                format_text(sig, chunk_ids, first_id + s0)
            raw = buf.view(torch.uint8)
            host = _pinned(slot, raw.numel())
            host.copy_(raw, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            if pending is not None:
                pending[1].synchronize()
                flush(pending[0])
            pending = (host, ev)
            slot ^= 1
            written += s1 - s0
        if pending is not None:
            pending[1].synchronize()
            flush(pending[0])
    return written


_WRITERS: list = []


def _pwrite_parallel(fd: int, mv: memoryview, offset: int, parts: int = 8, min_part: int = 4 << 20) -> None:
    import os
    from concurrent.futures import ThreadPoolExecutor

    n = len(mv)
    parts = max(1, min(parts, n // min_part))

    def put(k):
        lo, hi = n * k // parts, n * (k + 1) // parts
        while lo < hi:
            lo += os.pwritev(fd, [mv[lo:hi]], offset + lo)

    if parts == 1:
        put(0)
        return
    if not _WRITERS:
        _WRITERS.append(ThreadPoolExecutor(8))
    list(_WRITERS[0].map(put, range(parts)))
