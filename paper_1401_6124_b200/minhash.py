"""MinHash signatures and Jaccard estimation on B200 -- the drop-in API.

Mirrors ``minhashlab.minhash`` (reference minhash.py:1-206): ``FeatureSet``,
``Signature``, ``signature``, ``estimate_jaccard``, ``exact_jaccard`` and the
signature-file readers/writers keep the reference's names, argument meaning and
exceptions.  The per-set loop the reference runs on the CPU (kernels.py:21-73)
is replaced by the batched CSR kernels of libmhb (``signatures_csr``); the
per-set ``signature`` call is a batch of one.

There is no CPU path for signing: if libmhb.so or a CUDA device is missing,
the calls raise.
"""
from __future__ import annotations

import ctypes as C
import struct
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .families import Family, IterativeFamily, RandomFamily
from .modmath import MAX_KERNEL_PRIME


class FeatureSet:
    """Sorted, de-duplicated non-negative feature ids (reference minhash.py:21-62)."""

    __slots__ = ("ids",)

    def __init__(self, ids):
        if isinstance(ids, np.ndarray):
            arr = ids.astype(np.int64, copy=False)
        else:
            arr = np.array(list(ids), dtype=np.int64)
        arr = np.unique(arr)
        if arr.size and arr[0] < 0:
            raise ValueError("feature ids must be non-negative")
        arr.setflags(write=False)
        self.ids = arr

    def __len__(self) -> int:
        return int(self.ids.size)

    def __iter__(self):
        return iter(self.ids.tolist())

    def __eq__(self, other) -> bool:
        if not isinstance(other, FeatureSet):
            return NotImplemented
        return self.ids.shape == other.ids.shape and bool((self.ids == other.ids).all())

    def __hash__(self):
        return hash(self.ids.tobytes())

    def __repr__(self) -> str:
        return f"FeatureSet(size={len(self)})"

    @property
    def max_id(self) -> int:
        if self.ids.size == 0:
            raise ValueError("empty feature set has no max id")
        return int(self.ids[-1])


@dataclass(frozen=True, eq=False)
class Signature:
    """Per-hash argmin feature ids (int64, read-only) plus the family identity."""

    mins: np.ndarray
    family_key: tuple = field(default=())

    def __post_init__(self):
        arr = np.ascontiguousarray(self.mins, dtype=np.int64)
        arr.setflags(write=False)
        object.__setattr__(self, "mins", arr)

    def __len__(self) -> int:
        return int(self.mins.size)

    @classmethod
    def _wrap(cls, arr: np.ndarray, key: tuple) -> "Signature":
        """A Signature around a fresh contiguous int64 array (no copy, no checks)."""
        arr.setflags(write=False)
        obj = object.__new__(cls)
        object.__setattr__(obj, "mins", arr)
        object.__setattr__(obj, "family_key", key)
        return obj


def exact_jaccard(s1: FeatureSet, s2: FeatureSet) -> float:
    """|s1 & s2| / |s1 | s2|, 1.0 for two empty sets (reference minhash.py:81-88)."""
    x, y = s1.ids, s2.ids
    if x.size == 0 and y.size == 0:
        return 1.0
    inter = int(np.intersect1d(x, y, assume_unique=True).size)
    return inter / (int(x.size) + int(y.size) - inter)


# ---------------------------------------------------------------------------
# Batched CSR signing (the hot path)
# ---------------------------------------------------------------------------

def _torch():
    import torch

    return torch


MAX_ID = 2**32 - 1  # CSR feature ids are uint32


def _check_family(family: Family) -> None:
    if not isinstance(family, (IterativeFamily, RandomFamily)):
        raise TypeError(f"unsupported family type {type(family).__name__}")
    if family.prime >= 2**63:
        raise NotImplementedError(f"prime {family.prime} >= 2^63 is outside the reference's range too")


def _raise_status(status: int, family: Family) -> None:
    if status & _lib.STATUS_EMPTY_SET:
        raise ValueError("cannot build a signature for an empty feature set")
    if status & _lib.STATUS_ID_GE_PRIME:
        raise ValueError(f"feature id >= family prime {family.prime}")
    if status & _lib.STATUS_BAD_PARAM:
        raise ValueError("family parameters outside [1,p) x [0,p)")


def sign_csr_device(indptr, ids, family: Family, out, status=None, stream=None) -> None:
    """Raw asynchronous device call: indptr int64[S+1], ids uint32, out uint32/int64[S,N]
    CUDA tensors on one device.  No validation beyond the library's, no sync."""
    torch = _torch()
    sign_csr_to_ptr(indptr, ids, family, out.data_ptr(), out.dtype == torch.int64, status, stream)


class _Workspaces(threading.local):
    """Per-thread signing workspaces, one per (device, stream), grown on demand.  A
    workspace belongs to its launch stream (allocated on it, only ever used on it), so
    reuse across calls is stream-ordered; reuse saves an allocation per call, which
    matters for launch-bound small batches."""

    def __init__(self):
        self.by_stream = {}


_WS = _Workspaces()


def _workspace(dev, st, nbytes: int):
    torch = _torch()
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), st.cuda_stream)
    ws = _WS.by_stream.get(key)
    if ws is None or ws.numel() < nbytes:
        with torch.cuda.stream(st):
            ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _WS.by_stream[key] = ws
    return ws


def sign_csr_bands_device(indptr, ids, family: Family, rows_per_band: int, keys, out, status=None,
                          stream=None) -> None:
    """Raw asynchronous device call of the fused signing + band-key kernel
    (mhb_sign_iterative_csr_bands): out uint32/int64 [S, N] and keys uint64
    [S, N / rows_per_band] preallocated on the device.  No validation beyond the
    library's, no sync."""
    torch = _torch()
    lib = _lib.load()
    if not isinstance(family, IterativeFamily):
        raise TypeError("fused band keys need an iterative family")
    dev = ids.device
    n_sets = indptr.numel() - 1
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        ws_bytes = lib.mhb_sign_workspace_bytes(n_sets, ids.numel(), family.size)
        ws = _workspace(dev, st, ws_bytes)
        rc = lib.mhb_sign_iterative_csr_bands(
            indptr.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), family.base.a, family.base.b, family.prime,
            family.size, rows_per_band, keys.data_ptr(), out.data_ptr(),
            _lib.OUT_I64 if out.dtype == torch.int64 else _lib.OUT_U32, 1,
            status.data_ptr() if status is not None else None, ws.data_ptr(), ws_bytes, st.cuda_stream)
    _lib.check(rc)


def sign_csr_to_ptr(indptr, ids, family: Family, out_ptr: int, out_int64: bool = False, status=None,
                    stream=None) -> None:
    """sign_csr_device with the output given as a device address: rows [S, family.size]
    of uint32 (or int64) starting at `out_ptr` -- e.g. this rank's rows of a peer
    rank's matrix mapped with dist.PeerMatrix (fused sign + gather)."""
    torch = _torch()
    lib = _lib.load()
    dev = ids.device
    n_sets = indptr.numel() - 1
    nnz = ids.numel()
    n_hash = family.size
    out_dtype = _lib.OUT_I64 if out_int64 else _lib.OUT_U32
    ws_bytes = lib.mhb_sign_workspace_bytes(n_sets, nnz, n_hash)
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        sptr = st.cuda_stream
        ws = _workspace(dev, st, ws_bytes)
        status_ptr = status.data_ptr() if status is not None else None
        if isinstance(family, IterativeFamily):
            rc = lib.mhb_sign_iterative_csr(indptr.data_ptr(), ids.data_ptr(), n_sets, nnz,
                                            family.base.a, family.base.b, family.prime, n_hash,
                                            out_ptr, out_dtype, status_ptr,
                                            ws.data_ptr(), ws_bytes, sptr)
        elif family.prime > MAX_KERNEL_PRIME:
            a, b = family.device_params(dev, wide=True)
            rc = lib.mhb_sign_random_csr_u64(indptr.data_ptr(), ids.data_ptr(), n_sets, nnz,
                                             a.data_ptr(), b.data_ptr(), family.prime, n_hash,
                                             out_ptr, out_dtype, status_ptr, sptr)
        else:
            a, b = family.device_params(dev)
            rc = lib.mhb_sign_random_csr(indptr.data_ptr(), ids.data_ptr(), n_sets, nnz,
                                         a.data_ptr(), b.data_ptr(), family.prime, n_hash,
                                         out_ptr, out_dtype, status_ptr,
                                         ws.data_ptr(), ws_bytes, sptr)
    _lib.check(rc)


def signatures_csr(indptr, ids, family: Family, *, out_dtype="int64", out=None,
                   validate: bool = True, device=None):
    """Signatures of every set of a CSR batch.

    indptr: int64[S+1]; ids: feature ids (< family.prime), any order, repeats allowed.
    Device tensors in -> device tensor out (stream-ordered on the current stream;
    ``validate`` synchronises once to turn device status flags into the reference's
    ValueErrors).  numpy arrays in -> numpy array out through the host pipeline
    (mhb_sign_csr_host: chunked H2D / kernels / D2H overlap).
    Result: [S, family.size] argmin feature ids, int64 (reference dtype) or uint32.
    """
    _check_family(family)
    torch = _torch()
    if out_dtype not in ("int64", "uint32"):
        raise ValueError(f"out_dtype must be 'int64' or 'uint32', got {out_dtype!r}")
    if isinstance(ids, np.ndarray) or isinstance(indptr, np.ndarray):
        return _signatures_csr_host(np.asarray(indptr), np.asarray(ids), family, out_dtype, out, device)

    if not (ids.is_cuda and indptr.is_cuda):
        raise ValueError("signatures_csr needs CUDA tensors (or numpy arrays for the host pipeline)")
    if ids.dtype != torch.uint32:
        if ids.dtype in (torch.int64, torch.int32) and ids.numel():
            lo, hi = int(ids.min()), int(ids.max())
            if lo < 0:
                raise ValueError("feature ids must be non-negative")
            if hi >= family.prime:
                raise ValueError(f"feature id {hi} >= family prime {family.prime}")
            if hi > MAX_ID:  # the reference's int64 ids beyond 2^32 (primes >= 2^32)
                return _signatures_ids64(indptr, ids.to(torch.int64), family, out_dtype, out, validate)
        ids = ids.to(torch.uint32)
    ids = ids.contiguous()
    indptr = indptr.to(torch.int64).contiguous()
    n_sets = indptr.numel() - 1
    if validate and n_sets > 0:
        _check_indptr_device(indptr, ids.numel())
    tdt = torch.int64 if out_dtype == "int64" else torch.uint32
    if out is None:
        out = torch.empty((n_sets, family.size), dtype=tdt, device=ids.device)
    elif out.dtype != tdt or tuple(out.shape) != (n_sets, family.size) or not out.is_contiguous():
        raise ValueError("out has the wrong dtype, shape or layout")
    status = torch.zeros(1, dtype=torch.int32, device=ids.device) if validate else None
    sign_csr_device(indptr, ids, family, out, status)
    if validate:
        _raise_status(int(status.item()), family)
    return out


def _check_indptr_device(indptr, nnz: int) -> None:
    """ids are read at the absolute offsets indptr[s]: 0 <= indptr[0], indptr[-1] <= nnz and
    no decrease (one small device reduction and one read, before any launch)."""
    torch = _torch()
    bad = torch.stack([(indptr[0] < 0), (indptr[-1] > nnz), (indptr[1:] < indptr[:-1]).any()])
    flags = bad.cpu().tolist()
    if flags[0] or flags[1]:
        raise ValueError("indptr must satisfy 0 <= indptr[0] and indptr[-1] <= len(ids)")
    if flags[2]:
        raise ValueError("indptr must be non-decreasing")


def _signatures_ids64(indptr, ids, family: Family, out_dtype, out, validate):
    """Device CSR batch with int64 feature ids >= 2^32 (mhb_sign_csr_ids64, wide.cu)."""
    torch = _torch()
    if out_dtype != "int64":
        raise ValueError("feature ids >= 2^32 need out_dtype='int64'")
    lib = _lib.load()
    dev = ids.device
    indptr = indptr.to(torch.int64).contiguous()
    ids = ids.contiguous()
    n_sets = indptr.numel() - 1
    if out is None:
        out = torch.empty((n_sets, family.size), dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        sptr = torch.cuda.current_stream(dev).cuda_stream
        if isinstance(family, IterativeFamily):
            rc = lib.mhb_sign_csr_ids64(_lib.KIND_ITERATIVE, indptr.data_ptr(), ids.data_ptr(), n_sets, ids.numel(),
                                        family.base.a, family.base.b, None, None, family.prime, family.size,
                                        out.data_ptr(), status.data_ptr(), sptr)
        else:
            a, b = family.device_params(dev, wide=True)
            rc = lib.mhb_sign_csr_ids64(_lib.KIND_RANDOM, indptr.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), 0, 0,
                                        a.data_ptr(), b.data_ptr(), family.prime, family.size, out.data_ptr(),
                                        status.data_ptr(), sptr)
    _lib.check(rc)
    if validate:
        _raise_status(int(status.item()), family)
    return out


def _signatures_csr_host(indptr, ids, family, out_dtype, out, device):
    torch = _torch()
    lib = _lib.load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    if ids.dtype != np.uint32:
        if ids.size and (ids.min() < 0 or ids.max() >= family.prime or ids.max() > MAX_ID):
            if ids.min() < 0:
                raise ValueError("feature ids must be non-negative")
            if ids.max() >= family.prime:
                raise ValueError(f"feature id {int(ids.max())} >= family prime {family.prime}")
            # ids beyond 2^32 (primes >= 2^32): the 64-bit-id device entry
            dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
            res = _signatures_ids64(torch.as_tensor(indptr, device=dev), torch.as_tensor(ids.astype(np.int64), device=dev),
                                    family, out_dtype, None, True).cpu().numpy()
            if out is None:
                return res
            out[...] = res
            return out
        ids = ids.astype(np.uint32)
    if isinstance(family, RandomFamily) and family.prime > MAX_KERNEL_PRIME:
        # 64-bit random-family parameters: the device entry (mhb_sign_random_csr_u64)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        res = signatures_csr(torch.as_tensor(indptr, device=dev), torch.as_tensor(ids.astype(np.int64), device=dev),
                             family, out_dtype=out_dtype).cpu().numpy()
        if out is None:
            return res
        out[...] = res
        return out
    ids = np.ascontiguousarray(ids)
    n_sets = indptr.size - 1
    ndt = np.int64 if out_dtype == "int64" else np.uint32
    if out is None:
        out = np.empty((n_sets, family.size), dtype=ndt)
    elif out.dtype != ndt or out.shape != (n_sets, family.size) or not out.flags.c_contiguous:
        raise ValueError("out has the wrong dtype, shape or layout")
    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    status = C.c_int32(0)
    if isinstance(family, IterativeFamily):
        rc = lib.mhb_sign_csr_host(_lib.KIND_ITERATIVE, indptr.ctypes.data, ids.ctypes.data, n_sets, ids.size,
                                   family.base.a, family.base.b, None, None, family.prime, family.size,
                                   out.ctypes.data, _lib.OUT_I64 if ndt == np.int64 else _lib.OUT_U32,
                                   C.addressof(status), dev)
    else:
        a = np.ascontiguousarray(family.a, dtype=np.uint32)
        b = np.ascontiguousarray(family.b, dtype=np.uint32)
        rc = lib.mhb_sign_csr_host(_lib.KIND_RANDOM, indptr.ctypes.data, ids.ctypes.data, n_sets, ids.size,
                                   0, 0, a.ctypes.data, b.ctypes.data, family.prime, family.size,
                                   out.ctypes.data, _lib.OUT_I64 if ndt == np.int64 else _lib.OUT_U32,
                                   C.addressof(status), dev)
    _lib.check(rc)
    _raise_status(status.value, family)
    return out


def signature(s: FeatureSet, family: Family) -> Signature:
    """MinHash signature of one non-empty set (reference minhash.py:91-110): mins[i] is
    the feature id minimising h_i over s.  Runs the CUDA kernel on the current device."""
    ids = s.ids
    if ids.size == 0:
        raise ValueError("cannot build a signature for an empty feature set")
    max_id = int(ids[-1])  # canonical: sorted ascending
    if max_id >= family.prime:
        raise ValueError(f"feature id {max_id} >= family prime {family.prime}")
    if max_id > MAX_ID:  # int64 ids beyond 2^32: the 64-bit-id device entry
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device())
        ip = torch.tensor([0, len(s)], dtype=torch.int64, device=dev)
        out = _signatures_ids64(ip, torch.tensor(s.ids, device=dev), family, "int64", None, True)
        return Signature(out[0].cpu().numpy(), family.key)
    _check_family(family)
    if isinstance(family, RandomFamily) and family.prime > MAX_KERNEL_PRIME:  # 64-bit a, b: device entry
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device())
        dids = torch.from_numpy(ids.astype(np.uint32)).to(dev, non_blocking=False)
        indptr = torch.tensor([0, len(s)], dtype=torch.int64, device=dev)
        out = signatures_csr(indptr, dids, family, out_dtype="int64", validate=False)
        return Signature(out[0].cpu().numpy(), family.key)
    # host buffers -> mhb_sign_csr_host, whose small-batch path is served by the resident
    # doorbell block (csrc/small.cu); the FeatureSet is already canonical and checked above,
    # so the call goes straight through, staged in this thread's reusable buffers
    st = _PERSET
    n = int(ids.size)
    n_hash = family.size
    if n > st.ids.size or (n_hash < _PERSET_WIDE and n_hash > st.out.size):
        st.grow(n, n_hash)
    st.ids[:n] = ids  # int64 -> uint32 (ids < p < 2^32 checked above)
    st.indptr[1] = n
    if n_hash >= _PERSET_WIDE:
        # wide signatures (the reference's C6 loop: 100,000 hashes per call): a fresh result
        # the library fills in one copy (parallel above 256 KB), instead of a stage and two
        out, out_ptr = _perset_wide_result(n_hash)
    else:
        out, out_ptr = None, st.out_ptr
    kind, a, b, a_ptr, b_ptr = _percall_params(family)
    if out is not None and kind == _lib.KIND_RANDOM:  # wide random family: a, b already on the device
        da, db = family.device_params(_torch().device("cuda", _torch().cuda.current_device()))
        a_ptr, b_ptr = da.data_ptr(), db.data_ptr()
    rc = _sign_host()(kind, st.indptr_ptr, st.ids_ptr, 1, n, a, b, a_ptr, b_ptr, family.prime, n_hash, out_ptr,
                      _lib.OUT_I64, st.status_ptr, -1)
    if rc:
        _lib.check(rc)
    if st.status.value:
        _raise_status(st.status.value, family)
    return Signature._wrap(st.out[:n_hash].copy() if out is None else out, family.key)


_PERSET_WIDE = 8192  # per-set results at least this wide are written into a fresh array directly
# Wide results are page-locked (from torch's caching host allocator, already faulted in):
# the D2H lands in them directly, 54 vs 85 us per C6-shaped call against a fresh pageable
# array, whose first-touch page faults cost more than the copy.  Live page-locked results
# are capped (MHB_PERSET_PINNED_MB, default 1024) so retained signatures cannot pin
# unbounded host memory; beyond the cap results are ordinary arrays.
_PERSET_PINNED_CAP = int(__import__("os").environ.get("MHB_PERSET_PINNED_MB", "1024")) << 20
_perset_pinned = {"live": 0, "lock": threading.Lock()}


def _perset_unpin(nbytes: int) -> None:
    with _perset_pinned["lock"]:
        _perset_pinned["live"] -= nbytes


def _perset_wide_result(n_hash: int):
    nbytes = 8 * n_hash
    with _perset_pinned["lock"]:
        pin = _perset_pinned["live"] + nbytes <= _PERSET_PINNED_CAP
        if pin:
            _perset_pinned["live"] += nbytes
    if not pin:
        out = np.empty(n_hash, dtype=np.int64)
        return out, out.ctypes.data
    buf = _torch().empty(n_hash, dtype=_torch().int64, pin_memory=True)
    out = buf.numpy()
    weakref.finalize(out, _perset_unpin, nbytes)
    return out, buf.data_ptr()


class _PerSetStage(threading.local):
    """Per-thread reusable host buffers of the per-set API, their addresses taken once
    (numpy's .ctypes costs more than the GPU round trip of a small set)."""

    def __init__(self):
        self.indptr = np.zeros(2, dtype=np.int64)
        self.indptr_ptr = self.indptr.ctypes.data
        self.status = C.c_int32(0)
        self.status_ptr = C.addressof(self.status)
        self.ids = np.empty(0, dtype=np.uint32)
        self.out = np.empty(0, dtype=np.int64)
        self.ids_ptr = self.out_ptr = 0

    def grow(self, n: int, n_hash: int) -> None:
        if n > self.ids.size:
            self.ids = np.empty(max(n, 4096), dtype=np.uint32)
            self.ids_ptr = self.ids.ctypes.data
        if n_hash > self.out.size:
            self.out = np.empty(max(n_hash, 1024), dtype=np.int64)
            self.out_ptr = self.out.ctypes.data


_PERSET = _PerSetStage()
_SIGN_HOST = []


def _sign_host():
    """mhb_sign_csr_host, looked up once."""
    if not _SIGN_HOST:
        _SIGN_HOST.append(_lib.load().mhb_sign_csr_host)
    return _SIGN_HOST[0]


def _percall_params(family: Family) -> tuple:
    """(kind, a, b, a_host_ptr, b_host_ptr) of mhb_sign_csr_host for this family, built once."""
    hit = family.__dict__.get("_percall")
    if hit is None:
        if isinstance(family, IterativeFamily):
            hit = (_lib.KIND_ITERATIVE, family.base.a, family.base.b, None, None)
        else:
            a, b = family.host_params()  # cached on the family: the pointers stay valid
            hit = (_lib.KIND_RANDOM, 0, 0, a.ctypes.data, b.ctypes.data)
        family.__dict__["_percall"] = hit
    return hit


def signatures(sets, family: Family) -> list[Signature]:
    """Batch form of ``signature`` for a list of FeatureSets: one CSR launch."""
    sets = list(sets)
    if any(len(s) == 0 for s in sets):
        raise ValueError("cannot build a signature for an empty feature set")
    if not sets:
        return []
    sizes = np.array([len(s) for s in sets], dtype=np.int64)
    indptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ids = np.concatenate([s.ids for s in sets])
    if ids.max() >= family.prime:
        raise ValueError(f"feature id {int(ids.max())} >= family prime {family.prime}")
    # int64 ids as the FeatureSets hold them: signatures_csr narrows them to uint32 only
    # when they fit, and routes ids beyond 2^32 (primes >= 2^32) to the 64-bit-id entry
    mat = signatures_csr(indptr, ids, family, out_dtype="int64")
    return [Signature(row, family.key) for row in mat]


def estimate_jaccard(g1: Signature, g2: Signature) -> float:
    """Fraction of positions holding the same feature id (reference minhash.py:130-137)."""
    if g1.family_key != g2.family_key:
        raise ValueError(
            f"signatures come from different families: {g1.family_key} vs {g2.family_key}")
    if len(g1) != len(g2):
        raise ValueError("signature lengths differ")
    return float(np.mean(g1.mins == g2.mins))


def estimate_pairs(sig, pi, pj):
    """Jaccard estimates for listed pairs of rows of a device signature matrix.

    sig: CUDA [S, N] int64/uint32; pi, pj: int64 row indices.  Returns (counts uint32,
    estimates float64) where estimate = counts / N exactly as np.mean of the 0/1 vector
    (bench.py:165-168)."""
    torch = _torch()
    lib = _lib.load()
    pi = torch.as_tensor(pi, dtype=torch.int64, device=sig.device).contiguous()
    pj = torch.as_tensor(pj, dtype=torch.int64, device=sig.device).contiguous()
    n_pairs = pi.numel()
    if pj.numel() != n_pairs:
        raise ValueError("pair index arrays differ in length")
    counts = torch.empty(n_pairs, dtype=torch.uint32, device=sig.device)
    est = torch.empty(n_pairs, dtype=torch.float64, device=sig.device)
    dt = _lib.OUT_I64 if sig.dtype == torch.int64 else _lib.OUT_U32
    with torch.cuda.device(sig.device):
        rc = lib.mhb_jaccard_pairs(sig.data_ptr(), dt, sig.shape[1], pi.data_ptr(), pj.data_ptr(), n_pairs,
                                   counts.data_ptr(), est.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    return counts, est


def jaccard_block(sig_a, sig_b):
    """counts[r, c] = #{i : sig_a[r, i] == sig_b[c, i]} for two device signature blocks."""
    torch = _torch()
    lib = _lib.load()
    if sig_a.dtype != sig_b.dtype or sig_a.shape[1] != sig_b.shape[1]:
        raise ValueError("signature blocks differ in dtype or length")
    counts = torch.empty((sig_a.shape[0], sig_b.shape[0]), dtype=torch.uint32, device=sig_a.device)
    dt = _lib.OUT_I64 if sig_a.dtype == torch.int64 else _lib.OUT_U32
    with torch.cuda.device(sig_a.device):
        rc = lib.mhb_jaccard_block(sig_a.contiguous().data_ptr(), sig_a.shape[0], sig_b.contiguous().data_ptr(),
                                   sig_b.shape[0], dt, sig_a.shape[1], counts.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    return counts


def band_keys(sig, rows_per_band: int, *, keys=None, stream=None):
    """LSH band keys: uint64 [S, N/rows] from a device signature matrix [S, N].

    Bands are runs of `rows_per_band` consecutive hash positions; each key is
    splitmix64 of two polynomial hashes mod 2^32 over the band's argmin ids
    (include/mhb.h, csrc/bandhash.cuh).  Equal keys
    mean the two sets agree on every row of the band (the LSH candidate test).
    ``keys``: an optional preallocated uint64 [S, N/rows] output; ``stream``: the
    launch stream (default: the current one)."""
    torch = _torch()
    lib = _lib.load()
    n_sets, n_hash = sig.shape
    if n_hash % rows_per_band:
        raise ValueError(f"rows_per_band {rows_per_band} must divide the signature length {n_hash}")
    shape = (n_sets, n_hash // rows_per_band)
    if keys is None:
        keys = torch.empty(shape, dtype=torch.uint64, device=sig.device)
    elif keys.dtype != torch.uint64 or tuple(keys.shape) != shape or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous uint64 tensor of shape (n_sets, n_hash // rows_per_band)")
    dt = _lib.OUT_I64 if sig.dtype == torch.int64 else _lib.OUT_U32
    with torch.cuda.device(sig.device):
        st = stream if stream is not None else torch.cuda.current_stream()
        rc = lib.mhb_band_keys(sig.contiguous().data_ptr(), dt, n_sets, n_hash, rows_per_band, keys.data_ptr(),
                               st.cuda_stream)
    _lib.check(rc)
    return keys


def signatures_band_keys(indptr, ids, family: Family, rows_per_band: int, *, write_signatures: bool = True,
                         out_dtype: str = "uint32", validate: bool = True):
    """Signatures and their LSH band keys (device tensors).

    The keys are hashed inside the signing epilogue (mhb_sign_iterative_csr_bands,
    iterative family on the u32 kernels) when ``write_signatures=False`` (the matrix is
    never stored) or N >= 1024; otherwise the batch is signed and the standalone
    band-key kernel streams the matrix.  The keys always equal
    ``band_keys(signatures_csr(...), rows)``.
    """
    _check_family(family)
    torch = _torch()
    if rows_per_band <= 0 or family.size % rows_per_band:
        raise ValueError(f"rows_per_band {rows_per_band} must divide the signature length {family.size}")
    lanes = 64 if family.size >= 128 else 32  # the kernel's per-thread lane count K (sign.cu choose_geometry)
    # Keys only: fused into the signing epilogue (no signature matrix is written or re-read).
    # Signatures and keys: fused too for N >= 1024 (the skewed K = 64 kernels: cfg4 31.80 ms
    # against 34.33 ms for sign + the standalone key kernel, tools/bands_ab.py); below
    # that, sign, then the standalone key kernel, which streams the matrix at HBM speed
    # (cfg3 N = 512: 5.92 vs 6.49 ms fused).
    fusable = (isinstance(family, IterativeFamily) and family.prime <= MAX_KERNEL_PRIME and family.size >= 32
               and rows_per_band % 4 == 0 and lanes % rows_per_band == 0)
    fused = fusable and (not write_signatures or family.size >= 1024)
    if not fused or not (torch.is_tensor(ids) and ids.is_cuda):
        sig = signatures_csr(indptr, ids, family, out_dtype=out_dtype, validate=validate)
        if not torch.is_tensor(sig):
            sig = torch.from_numpy(sig).cuda()
        keys = band_keys(sig, rows_per_band)
        return (sig if write_signatures else None), keys
    if ids.dtype != torch.uint32:
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= family.prime):
            raise ValueError("feature ids must be in [0, family.prime)")
        ids = ids.to(torch.uint32)
    ids = ids.contiguous()
    indptr = indptr.to(torch.int64).contiguous()
    n_sets = indptr.numel() - 1
    if validate and n_sets > 0:
        _check_indptr_device(indptr, ids.numel())
    tdt = torch.int64 if out_dtype == "int64" else torch.uint32
    lib = _lib.load()
    dev = ids.device
    sig = torch.empty((n_sets, family.size), dtype=tdt, device=dev)
    keys = torch.empty((n_sets, family.size // rows_per_band), dtype=torch.uint64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev) if validate else None
    ws_bytes = lib.mhb_sign_workspace_bytes(n_sets, ids.numel(), family.size)
    with torch.cuda.device(dev):
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        rc = lib.mhb_sign_iterative_csr_bands(
            indptr.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), family.base.a, family.base.b, family.prime,
            family.size, rows_per_band, keys.data_ptr(), sig.data_ptr(),
            _lib.OUT_I64 if tdt == torch.int64 else _lib.OUT_U32, 1 if write_signatures else 0,
            status.data_ptr() if status is not None else None, ws.data_ptr(), ws_bytes,
            torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc)
    if validate:
        _raise_status(int(status.item()), family)
    return (sig if write_signatures else None), keys


# ---------------------------------------------------------------------------
# Signature files (reference minhash.py:140-206): "id N ids..." text lines and
# little-endian u64 binary records.
# ---------------------------------------------------------------------------

def _record_mins(sig) -> np.ndarray:
    mins = sig.mins if isinstance(sig, Signature) else np.asarray(sig, dtype=np.int64)
    if mins.ndim != 1:
        raise ValueError("signature record must be a 1-d id vector")
    return mins


def write_signatures_text(path, records) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for obj_id, sig in records:
            mins = _record_mins(sig)
            fh.write(f"{int(obj_id)} {mins.size} " + " ".join(map(str, mins.tolist())) + "\n")


def read_signatures_text(path) -> list[tuple[int, np.ndarray]]:
    records = []
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            fields = line.split()
            if not fields:
                continue
            if len(fields) < 2:
                raise ValueError(f"{path}:{lineno}: truncated signature record")
            obj_id, n = int(fields[0]), int(fields[1])
            ids = np.array([int(v) for v in fields[2:]], dtype=np.int64)
            if ids.size != n:
                raise ValueError(f"{path}:{lineno}: record declares {n} ids but carries {ids.size}")
            records.append((obj_id, ids))
    return records


def write_signatures_binary(path, records) -> None:
    with open(path, "wb") as fh:
        for obj_id, sig in records:
            mins = _record_mins(sig)
            fh.write(struct.pack("<QQ", int(obj_id), mins.size))
            fh.write(mins.astype("<u8").tobytes())


def read_signatures_binary(path) -> list[tuple[int, np.ndarray]]:
    records = []
    with open(path, "rb") as fh:
        while True:
            head = fh.read(16)
            if not head:
                break
            if len(head) < 16:
                raise ValueError(f"{path}: truncated record header")
            obj_id, n = struct.unpack("<QQ", head)
            body = fh.read(8 * n)
            if len(body) < 8 * n:
                raise ValueError(f"{path}: truncated record body")
            records.append((int(obj_id), np.frombuffer(body, dtype="<u8").astype(np.int64)))
    return records
