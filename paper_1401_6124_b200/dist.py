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
    `align` (align=2 keeps planted pairs (2k, 2k+1) on one rank).  A device indptr
    is searched on the device: only the world-1 cut points come back to the host."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if hasattr(indptr, "is_cuda") and indptr.is_cuda:
        import torch

        n_sets = indptr.numel() - 1
        ends = indptr[[0, -1]].cpu().tolist()
        base, total = int(ends[0]), int(ends[1] - ends[0])
        goals = torch.tensor([base + (total * r) // world for r in range(1, world)], dtype=torch.int64,
                             device=indptr.device)
        raw = torch.searchsorted(indptr.contiguous(), goals, side="left").cpu().tolist() if world > 1 else []
    else:
        ip = np.asarray(indptr.cpu() if hasattr(indptr, "cpu") else indptr, dtype=np.int64)
        n_sets = ip.size - 1
        base, total = int(ip[0]), int(ip[-1] - ip[0])
        raw = [int(np.searchsorted(ip, base + (total * r) // world, side="left")) for r in range(1, world)]
    cuts = [0]
    for c in raw:
        c = min(max(int(c), cuts[-1]), n_sets)
        c -= c % align
        cuts.append(max(c, cuts[-1]))
    cuts.append(n_sets)
    return cuts


def shard_of(indptr, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    cuts = nnz_balanced_cuts(indptr, world, align)
    return cuts[rank], cuts[rank + 1]


def _flag_device(group=None):
    """Where this process group's collectives take their tensors (NCCL: the current GPU)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def agree_or_raise(err: BaseException | None, group=None, what: str = "signing") -> None:
    """Collective error check: every rank reaches it, learns whether ANY rank failed,
    and all raise together -- so no rank is left waiting in a later barrier or gather."""
    import torch
    import torch.distributed as dist

    flag = torch.tensor([1 if err is not None else 0], dtype=torch.int32, device=_flag_device(group))
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if err is not None:
        raise err
    if int(flag.item()):
        raise RuntimeError(f"{what} failed on another rank")


def _default_sign(indptr, ids, family):
    """This rank's rows with the library's checks: the reference's ValueErrors for empty
    sets and ids >= p (status word), ids outside uint32 rejected before the cast."""
    import torch

    from .minhash import signatures_csr

    if indptr.numel() - 1 == 0:
        return torch.empty((0, family.size), dtype=torch.uint32, device=ids.device)
    return signatures_csr(indptr, ids, family, out_dtype="uint32", validate=True)


def _slice_shard(indptr, ids, s0: int, s1: int, device):
    """Rows [s0, s1) of a global CSR batch as (indptr from 0, ids) on `device`.  Device
    tensors are sliced in place (views; no host round trip); host arrays copy only the
    slice."""
    import torch

    if torch.is_tensor(indptr) and indptr.is_cuda:
        lo, hi = (int(v) for v in indptr[[s0, s1]].cpu().tolist())
        ip = indptr[s0:s1 + 1] - lo
    else:
        ip_h = np.asarray(indptr.cpu() if hasattr(indptr, "cpu") else indptr, dtype=np.int64)
        lo, hi = int(ip_h[s0]), int(ip_h[s1])
        ip = torch.as_tensor(ip_h[s0:s1 + 1] - lo)
    if torch.is_tensor(ids):
        x = ids[lo:hi]
    else:
        x = torch.as_tensor(np.ascontiguousarray(np.asarray(ids)[lo:hi]))
    if device is not None:
        ip, x = ip.to(device), x.to(device)
    return ip.contiguous(), x.contiguous()


def gather_blocks(block, rows_per_rank: list[int], dst: int = 0, group=None):
    """Gather variable-height [rows, N] blocks to `dst` with no padding: `dst` allocates
    the [sum(rows), N] matrix and receives every other rank's block straight into its
    row range (point-to-point; one NCCL group on the GPU backend).  Returns the matrix
    on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if len(rows_per_rank) != world:
        raise ValueError("rows_per_rank needs one entry per rank")
    if block.shape[0] != rows_per_rank[rank]:
        raise ValueError(f"rank {rank} holds {block.shape[0]} rows, rows_per_rank says {rows_per_rank[rank]}")
    n = block.shape[1]
    is_u32 = block.dtype == torch.uint32
    wire = block.view(torch.int32) if is_u32 else block
    nccl = dist.get_backend(group) == "nccl"
    g = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    if rank == dst:
        full = torch.empty((sum(rows_per_rank), n), dtype=wire.dtype, device=block.device)
        off = 0
        ops, works = [], []
        for r, h in enumerate(rows_per_rank):
            part = full[off:off + h]
            off += h
            if r == rank:
                part.copy_(wire)
            elif h > 0:
                if nccl:
                    ops.append(dist.P2POp(dist.irecv, part, g(r), group))
                else:
                    works.append(dist.irecv(part, src=g(r), group=group))
        if ops:
            works += dist.batch_isend_irecv(ops)
        for w in works:
            w.wait()
        return full.view(torch.uint32) if is_u32 else full
    if rows_per_rank[rank] > 0:
        if nccl:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, wire.contiguous(), g(dst), group)]):
                w.wait()
        else:
            dist.send(wire.contiguous(), dst=g(dst), group=group)
    return None


def sign_sharded(indptr, ids, family, *, sign_fn=None, gather: bool = True, dst: int = 0,
                 align: int = 1, device=None, group=None):
    """Sign this rank's nnz-balanced slice of a global CSR batch.

    indptr/ids: the global batch -- device tensors (sliced in place, nothing copied to
    the host) or host arrays (only this rank's slice is copied).  Every rank sees the
    same batch and derives the same cuts.  Errors on any rank (an empty set, an id >= p)
    raise on every rank before the gather.  Returns (local_block, (s0, s1), full) where
    full is the gathered [S, N] matrix on `dst` when gather=True, else None."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    cuts = nnz_balanced_cuts(indptr, world, align)
    s0, s1 = cuts[rank], cuts[rank + 1]
    block, err = None, None
    try:
        local_ip, local_ids = _slice_shard(indptr, ids, s0, s1, device)
        block = (sign_fn or _default_sign)(local_ip, local_ids, family)
    except Exception as e:  # noqa: BLE001 -- re-raised below, on every rank together
        err = e
    agree_or_raise(err, group)
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
    kernels complete (stream sync) before the barrier that publishes the matrix.  The
    reference's input errors (empty set, id >= p) raise on every rank together, and
    every rank passes the same barriers whatever happens."""
    import torch
    import torch.distributed as dist

    from .minhash import _check_indptr_device, _raise_status, sign_csr_to_ptr

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    cuts = nnz_balanced_cuts(indptr, world, align)
    s0, s1 = cuts[rank], cuts[rank + 1]
    n_total = cuts[-1]
    err, local_ip, local_ids = None, None, None
    try:
        local_ip, local_ids = _slice_shard(indptr, ids, s0, s1, dev)
        if local_ids.dtype != torch.uint32:
            if local_ids.numel() and (int(local_ids.min()) < 0 or int(local_ids.max()) >= family.prime):
                raise ValueError(f"feature ids must be in [0, family.prime = {family.prime})")
            local_ids = local_ids.to(torch.int64).to(torch.uint32)
        if s1 > s0:
            _check_indptr_device(local_ip, local_ids.numel())
    except Exception as e:  # noqa: BLE001
        err = e
    agree_or_raise(err, group, "input checks")
    mat = PeerMatrix.allocate(n_total, family.size, 4, dev.index) if rank == dst else None
    box = [mat.handle if mat is not None else None]
    dist.broadcast_object_list(box, src=dst, group=group)
    view = mat if rank == dst else PeerMatrix.open(box[0], n_total, family.size, 4, dev.index)
    err = None
    try:
        if s1 > s0:
            status = torch.zeros(1, dtype=torch.int32, device=dev)
            sign_csr_to_ptr(local_ip, local_ids, family, view.ptr(s0), False, status)
            _raise_status(int(status.item()), family)
        torch.cuda.synchronize(dev)
    except Exception as e:  # noqa: BLE001
        err = e
    try:
        agree_or_raise(err, group)  # doubles as the barrier: every row has landed in dst's matrix
    except BaseException:
        if rank != dst:
            view.close()
        dist.barrier(group=group)
        if mat is not None:
            mat.close()
        raise
    if rank != dst:
        view.close()
    dist.barrier(group=group)  # every mapping is closed before dst may free the matrix
    return (mat if rank == dst else None), (s0, s1)
