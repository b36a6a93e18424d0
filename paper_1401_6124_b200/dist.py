"""Row-sharded multi-GPU signing: nnz-balanced partition + gather (NCCL, or fused over peer memory).

Sets are independent (reference minhash.py:91-110 signs one set at a time), so
the batch shards by rows with no exchange during compute.  Every rank derives
the same cut points from indptr alone -- no communication -- and rebuilds the
family from (kind, seed, hashes, prime) (families.py:236-259), so nothing is
broadcast either (the paper's MapReduce remark).  The only
collective is the optional gather of uint32 signature blocks to one rank.

One process per GPU (torchrun); ``torch.distributed`` with backend "nccl" on the
box, "gloo" in the CPU tests (which inject the CPU oracle as ``sign_fn``).

Fused sign + gather (``sign_gather_peer``): the destination rank allocates the
full [S, N] matrix as a ``PeerMatrix`` (CUDA IPC handle, csrc/peer.cu), every rank
maps it and signs its rows straight into it -- the kernels' epilogue stores cross
NVLink tile by tile while the rest of the shard is still being signed, so there is
no separate gather step.  The handle travels once over the process group.
"""
from __future__ import annotations

import numpy as np


def nnz_balanced_cuts(indptr, world: int, align: int = 1) -> list[int]:
    """Set boundaries [0, c_1, ..., c_{world-1}, S] with ~equal nnz per range.

    c_r = searchsorted(indptr, r * nnz / world) rounded down to a multiple of
    `align` (align=2 keeps planted pairs (2k, 2k+1) on one rank)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    ip = np.asarray(indptr.cpu() if hasattr(indptr, "cpu") else indptr, dtype=np.int64)
    n_sets = ip.size - 1
    base, total = int(ip[0]), int(ip[-1] - ip[0])
    cuts = [0]
    for r in range(1, world):
        goal = base + (total * r) // world
        c = int(np.searchsorted(ip, goal, side="left"))
        c = min(max(c, cuts[-1]), n_sets)
        c -= c % align
        cuts.append(max(c, cuts[-1]))
    cuts.append(n_sets)
    return cuts


def shard_of(indptr, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    cuts = nnz_balanced_cuts(indptr, world, align)
    return cuts[rank], cuts[rank + 1]


def _default_sign(indptr, ids, family):
    import torch

    from .minhash import sign_csr_device

    out = torch.empty((indptr.numel() - 1, family.size), dtype=torch.uint32, device=ids.device)
    if out.shape[0]:
        sign_csr_device(indptr, ids, family, out)
    return out


def gather_blocks(block, rows_per_rank: list[int], dst: int = 0, group=None):
    """Gather variable-height [rows, N] blocks to `dst` (padded to the max height on
    the wire, trimmed on arrival).  Returns the stacked matrix on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = block.shape[1]
    hmax = max(rows_per_rank) if rows_per_rank else 0
    wire_dtype = torch.int32 if block.dtype == torch.uint32 else block.dtype
    send = torch.zeros((hmax, n), dtype=wire_dtype, device=block.device)
    if block.shape[0]:
        send[:block.shape[0]].copy_(block.view(wire_dtype) if block.dtype == torch.uint32 else block)
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, gather_list=bufs, dst=dst, group=group)
    if rank != dst:
        return None
    parts = [b[:h] for b, h in zip(bufs, rows_per_rank)]
    full = torch.cat(parts, 0)
    return full.view(torch.uint32) if block.dtype == torch.uint32 else full


def sign_sharded(indptr, ids, family, *, sign_fn=None, gather: bool = True, dst: int = 0,
                 align: int = 1, device=None, group=None):
    """Sign this rank's nnz-balanced slice of a global CSR batch.

    indptr/ids: the global batch (host numpy or torch; every rank sees the same
    arrays).  Returns (local_block, (s0, s1), full) where full is the gathered
    [S, N] matrix on `dst` when gather=True, else None."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    cuts = nnz_balanced_cuts(indptr, world, align)
    s0, s1 = cuts[rank], cuts[rank + 1]
    ip = torch.as_tensor(np.asarray(indptr.cpu() if hasattr(indptr, "cpu") else indptr, dtype=np.int64))
    lo, hi = int(ip[s0]), int(ip[s1])
    ids_t = torch.as_tensor(ids.cpu().numpy() if hasattr(ids, "cpu") else np.asarray(ids))
    local_ip = (ip[s0:s1 + 1] - lo).clone()
    local_ids = ids_t[lo:hi].clone()
    if device is not None:
        local_ip = local_ip.to(device)
        local_ids = local_ids.to(device)
    fn = sign_fn or _default_sign
    block = fn(local_ip, local_ids, family)
    full = None
    if gather:
        rows = [cuts[r + 1] - cuts[r] for r in range(world)]
        full = gather_blocks(block, rows, dst=dst, group=group)
    return block, (s0, s1), full


class PeerMatrix:
    """A [rows, cols] uint32/int64 device matrix shared across processes (csrc/peer.cu).

    The owner allocates it (``PeerMatrix.allocate``) and passes ``handle`` (64 bytes)
    to the others, which map it (``PeerMatrix.open``).  ``ptr(row)`` is the device
    address of a row in this process's mapping; ``tensor()`` views the mapping as a
    torch tensor.  ``close()`` unmaps / frees."""

    def __init__(self, ptr: int, handle: bytes, rows: int, cols: int, itemsize: int, owner: bool, device: int):
        self._ptr, self.handle, self.rows, self.cols = ptr, handle, rows, cols
        self.itemsize, self.owner, self.device = itemsize, owner, device

    @classmethod
    def allocate(cls, rows: int, cols: int, itemsize: int = 4, device: int = 0) -> "PeerMatrix":
        import ctypes as C

        from . import _lib

        lib = _lib.load()
        ptr, h = C.c_void_p(), (C.c_ubyte * 64)()
        _lib.check(lib.mhb_peer_alloc(rows * cols * itemsize, device, C.byref(ptr), h))
        return cls(ptr.value, bytes(h), rows, cols, itemsize, True, device)

    @classmethod
    def open(cls, handle: bytes, rows: int, cols: int, itemsize: int = 4, device: int = 0) -> "PeerMatrix":
        import ctypes as C

        from . import _lib

        lib = _lib.load()
        ptr = C.c_void_p()
        h = (C.c_ubyte * 64).from_buffer_copy(handle)
        _lib.check(lib.mhb_peer_open(h, device, C.byref(ptr)))
        return cls(ptr.value, handle, rows, cols, itemsize, False, device)

    def ptr(self, row: int = 0) -> int:
        return self._ptr + row * self.cols * self.itemsize

    @property
    def __cuda_array_interface__(self):
        typestr = "<u4" if self.itemsize == 4 else "<i8"
        return {"shape": (self.rows, self.cols), "typestr": typestr, "data": (self._ptr, False), "version": 3}

    def tensor(self):
        """Zero-copy torch view of this process's mapping (keeps this object alive;
        invalid after close())."""
        import torch

        if not self._ptr:
            raise RuntimeError("the matrix is closed")
        return torch.as_tensor(self, device=f"cuda:{self.device}")

    def close(self) -> None:
        from . import _lib

        if self._ptr:
            lib = _lib.load()
            _lib.check(lib.mhb_peer_free(self._ptr) if self.owner else lib.mhb_peer_close(self._ptr))
            self._ptr = 0


def sign_gather_peer(indptr, ids, family, *, dst: int = 0, align: int = 1, device=None, group=None):
    """Fused sign + gather: every rank signs its nnz-balanced slice directly into the
    destination rank's [S, N] uint32 matrix (mapped over CUDA IPC / NVLink).

    Returns (matrix, (s0, s1)): on `dst` the PeerMatrix holding every signature
    (``.tensor()`` views it; the caller closes it), elsewhere None.  Each rank's
    kernels complete (stream sync) before the barrier that publishes the matrix."""
    import torch
    import torch.distributed as dist

    from .minhash import sign_csr_to_ptr

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    cuts = nnz_balanced_cuts(indptr, world, align)
    s0, s1 = cuts[rank], cuts[rank + 1]
    n_total = cuts[-1]
    ip = np.asarray(indptr.cpu() if hasattr(indptr, "cpu") else indptr, dtype=np.int64)
    lo, hi = int(ip[s0]), int(ip[s1])
    local_ip = torch.as_tensor(ip[s0:s1 + 1] - lo).to(dev)
    x = ids if torch.is_tensor(ids) else torch.from_numpy(np.asarray(ids))
    local_ids = x[lo:hi].to(dev)
    if local_ids.dtype != torch.uint32:
        local_ids = local_ids.to(torch.int64).to(torch.uint32)
    mat = PeerMatrix.allocate(n_total, family.size, 4, dev.index) if rank == dst else None
    box = [mat.handle if mat is not None else None]
    dist.broadcast_object_list(box, src=dst, group=group)
    view = mat if rank == dst else PeerMatrix.open(box[0], n_total, family.size, 4, dev.index)
    try:
        if s1 > s0:
            sign_csr_to_ptr(local_ip, local_ids, family, view.ptr(s0))
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)  # every row has landed in dst's matrix
    finally:
        if rank != dst:
            view.close()
    dist.barrier(group=group)  # every mapping is closed before dst may free the matrix
    return (mat if rank == dst else None), (s0, s1)
