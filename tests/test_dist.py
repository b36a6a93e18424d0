"""Multi-rank sharding and gather, exercised with the gloo backend on CPU.

The product path runs one process per GPU over NCCL; here two CPU ranks run the
same driver (paper_1401_6124_b200.dist) with the CPU oracle injected as the
per-shard signer, and rank 0 checks the gathered matrix against the oracle on
the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1401_6124_b200 import gen, make_family
from paper_1401_6124_b200.dist import nnz_balanced_cuts, shard_of


def test_cuts_balance_nnz():
    rng = np.random.default_rng(1)
    sizes = rng.integers(1, 400, size=5000)
    ip = np.concatenate([[0], np.cumsum(sizes)])
    for world in (1, 2, 3, 8):
        cuts = nnz_balanced_cuts(ip, world)
        assert cuts[0] == 0 and cuts[-1] == 5000 and all(a <= b for a, b in zip(cuts, cuts[1:]))
        loads = [ip[cuts[r + 1]] - ip[cuts[r]] for r in range(world)]
        assert max(loads) - min(loads) <= 2 * sizes.max()


def test_cuts_keep_pairs_together():
    ip = np.arange(0, 1001 * 3, 3)
    for world in (2, 4, 7):
        cuts = nnz_balanced_cuts(ip, world, align=2)
        assert all(c % 2 == 0 for c in cuts[:-1])
    assert shard_of(ip, 0, 1) == (0, 1000)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_1401_6124_b200.dist import sign_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        indptr, ids = gen.cfg1_numpy(n_sets=333, seed=11)
        fam = make_family("iterative", 7, 64, 1_048_583)

        def sign_fn(ip, x, family):
            out = oracle.sign_family_csr(ip.numpy(), x.numpy().astype(np.uint32), family)
            return torch.from_numpy(out.astype(np.int32)).view(torch.uint32)

        block, (s0, s1), full = sign_sharded(indptr, ids, fam, sign_fn=sign_fn)
        if rank == 0:
            want = oracle.sign_family_csr(indptr, ids, fam)
            q.put(bool(np.array_equal(full.view(torch.int32).numpy().astype(np.int64), want)))
        else:
            q.put(full is None and block.shape[0] == s1 - s0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_sign_and_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(results) and all(p.exitcode == 0 for p in procs)


def _split_worker(rank, world, port, q):
    """The north-star split on CPU: every rank rebuilds the global indptr of one blocked
    batch, cuts it, generates only its own shard, signs it (oracle as the signer) and
    gathers unpadded blocks; rank 0 compares with the whole batch generated in one piece."""
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_1401_6124_b200.dist import gather_blocks, nnz_balanced_cuts

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = gen.CONFIGS["cfg2"]
        n = 3000
        ip_g = gen.global_indptr(cfg, "cpu", n, block=700)
        cuts = nnz_balanced_cuts(ip_g, world)
        s0, s1 = cuts[rank], cuts[rank + 1]
        ip, ids, _ = gen.make_shard(cfg, s0, s1, "cpu", n, block=700, indptr=ip_g)
        fam = make_family("iterative", 3, 64, cfg.prime)
        blk = oracle.sign_family_csr(ip.numpy(), ids.numpy().view(np.uint32), fam).astype(np.uint32)
        full = gather_blocks(torch.from_numpy(blk.view(np.int32)).view(torch.uint32),
                             [cuts[r + 1] - cuts[r] for r in range(world)])
        if rank == 0:
            ip1, ids1, _ = gen.make_shard(cfg, 0, n, "cpu", n, block=700)
            want = oracle.sign_family_csr(ip1.numpy(), ids1.numpy().view(np.uint32), fam)
            q.put(bool(np.array_equal(full.view(torch.int32).numpy().astype(np.int64), want)))
        else:
            q.put(full is None)
    finally:
        dist.destroy_process_group()


def _error_worker(rank, world, port, q):
    """A data error on ONE rank (an id >= p) raises on every rank before the gather --
    nobody is left waiting in a collective."""
    import torch
    import torch.distributed as dist

    from paper_1401_6124_b200.dist import sign_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        indptr, ids = gen.cfg1_numpy(n_sets=200, seed=2)
        fam = make_family("iterative", 7, 32, 1_048_583)

        def sign_fn(ip, x, family):
            if int(x.to(torch.int64).max()) >= family.prime or dist.get_rank() == 1:
                raise ValueError("feature id >= family prime")
            return torch.zeros((ip.numel() - 1, family.size), dtype=torch.int32).view(torch.uint32)

        try:
            sign_sharded(indptr, ids, fam, sign_fn=sign_fn)
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, "ValueError"))
        except RuntimeError as e:
            q.put((rank, "RuntimeError"))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return results, procs


def test_gloo_split_of_one_global_batch():
    results, procs = _spawn(_split_worker, 2)
    assert all(results) and all(p.exitcode == 0 for p in procs)


def test_gloo_error_on_one_rank_raises_everywhere():
    results, procs = _spawn(_error_worker, 2)
    got = dict(results)
    assert got == {0: "RuntimeError", 1: "ValueError"}, got
    assert all(p.exitcode == 0 for p in procs)


def test_gen_shards_concatenate_to_the_batch():
    import torch

    for name, n, block in (("cfg2", 2500, 600), ("cfg3", 2400, 300), ("cfg5", 1800, 500)):
        cfg = gen.CONFIGS[name]
        ip_g = gen.global_indptr(cfg, "cpu", n, block=block)
        whole = gen.make_shard(cfg, 0, n, "cpu", n, block=block, indptr=ip_g)
        for world in (2, 3):
            cuts = nnz_balanced_cuts(ip_g, world, align=2 if name == "cfg3" else 1)
            parts = [gen.make_shard(cfg, cuts[r], cuts[r + 1], "cpu", n, block=block, indptr=ip_g)
                     for r in range(world)]
            assert torch.equal(torch.cat([p[1] for p in parts]), whole[1])
            if name == "cfg3":
                assert torch.equal(torch.cat([p[2] for p in parts]), whole[2])
