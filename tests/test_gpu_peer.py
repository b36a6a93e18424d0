"""Fused sign + gather over peer memory (dist.sign_gather_peer, csrc/peer.cu).

Every rank maps the destination rank's [S, N] matrix through a CUDA IPC handle and
its signing kernels store their rows straight into it.  The box has one GPU, so the
ranks here are processes sharing cuda:0 (same-device IPC): the code path -- handle
export/import, per-rank row offsets, long-set red.global.min merges and finalize on
mapped memory, the publish/unmap barriers -- is the multi-GPU one; the kernels never
wait on each other (only host barriers after completion).  Result: bit-exact
against the single-process signatures of the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch():
    from paper_1401_6124_b200 import gen

    indptr, ids = gen.cfg1_numpy(n_sets=3000, seed=9)
    rng = np.random.default_rng(4)
    rows = [ids[indptr[s]:indptr[s + 1]] for s in range(indptr.size - 1)]
    for n in (1500, 5000):  # long sets: chunk merges into the mapped matrix
        rows.insert(int(rng.integers(0, len(rows))), rng.choice(1 << 20, size=n, replace=False).astype(np.uint32))
    ip = np.zeros(len(rows) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([r.size for r in rows])
    return ip, np.concatenate(rows).astype(np.uint32)


def _worker(rank, world, port, kind, q):
    import torch
    import torch.distributed as dist

    from paper_1401_6124_b200 import make_family, signatures_csr
    from paper_1401_6124_b200.dist import sign_gather_peer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ip, ids = _batch()
        fam = make_family(kind, 5, 256, 1_048_583)
        mat, (s0, s1) = sign_gather_peer(ip, ids, fam, device="cuda:0")
        if rank == 0:
            got = mat.tensor().cpu().numpy().copy()
            mat.close()
            want = signatures_csr(torch.as_tensor(ip, device="cuda:0"),
                                  torch.as_tensor(ids.astype(np.int64), device="cuda:0").to(torch.uint32),
                                  fam, out_dtype="uint32").cpu().numpy()
            q.put(("ok", bool(np.array_equal(got, want)), int((got != want).sum())))
    except Exception as exc:  # surface the failure to the parent
        q.put(("error", repr(exc), 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "iterative"), (3, "random")])
def test_sign_gather_peer_matches_single_process(cuda_device, world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), kind, q), nprocs=world, join=True,
                       start_method="spawn")
    status, equal, n_diff = q.get(timeout=60)
    assert status == "ok", equal
    assert equal, f"{n_diff} entries differ"


def test_peer_matrix_single_rank(cuda_device):
    """world == 1: the owner signs into its own PeerMatrix (no mapping)."""
    import torch

    from paper_1401_6124_b200 import make_family, signatures_csr
    from paper_1401_6124_b200.dist import PeerMatrix
    from paper_1401_6124_b200.minhash import sign_csr_to_ptr

    ip, ids = _batch()
    fam = make_family("iterative", 2, 128, 1_048_583)
    m = PeerMatrix.allocate(ip.size - 1, 128, 4, 0)
    try:
        dip = torch.as_tensor(ip, device="cuda:0")
        dids = torch.as_tensor(ids.astype(np.int64), device="cuda:0").to(torch.uint32)
        sign_csr_to_ptr(dip, dids, fam, m.ptr(0))
        torch.cuda.synchronize()
        want = signatures_csr(dip, dids, fam, out_dtype="uint32")
        assert torch.equal(m.tensor().view(torch.int32), want.view(torch.int32))
    finally:
        m.close()


def test_bench_two_ranks_on_one_gpu():
    """bench.py's N>1 path -- one global batch cut into nnz-balanced shards, each rank
    generating only its own shard, barriers, max over ranks, the variable-size gather
    and the fused peer gather with every rank checking its rows -- with both ranks on
    the box's one GPU over gloo (MHB_BENCH_SHARED_GPU=1).  Checks the plumbing, not the
    timings."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, MHB_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "cfg2", "--n-sets", "50000", "--gather", "auto", "--no-cpu-baseline", "--e2e-steps", "1"]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "strong"
    assert line["config"]["n_sets"] == 50000
    g = line["gather"]
    assert not any(k.endswith("error") for k in g), g
    assert g["bytes_to_rank0_per_step"] == 50000 * 256 * 4
    assert g["nccl"]["ms"] > 0 and g["peer"]["ms_per_step"] > 0
    assert line["e2e"]["sets_per_step"] > 0 and line["e2e_reference_convention"]["value"] > 0


def _shard_worker(rank, world, port, cfg_name, n_sets, q):
    """One rank of the north-star split: global indptr -> cuts -> own shard -> sign ->
    unpadded gather to rank 0, which compares with the single-process signatures of
    the same global batch."""
    import torch
    import torch.distributed as dist

    from paper_1401_6124_b200 import gen, make_family, signatures_csr
    from paper_1401_6124_b200.dist import gather_blocks, nnz_balanced_cuts

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = gen.CONFIGS[cfg_name]
        dev = torch.device("cuda", 0)
        ip_g = gen.global_indptr(cfg, dev, n_sets)
        cuts = nnz_balanced_cuts(ip_g, world, align=2 if cfg_name == "cfg3" else 1)
        s0, s1 = cuts[rank], cuts[rank + 1]
        ip, ids, _ = gen.make_shard(cfg, s0, s1, dev, n_sets, indptr=ip_g)
        fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
        block = signatures_csr(ip, ids, fam, out_dtype="uint32")
        full = gather_blocks(block.cpu(), [cuts[r + 1] - cuts[r] for r in range(world)], dst=0)
        if rank == 0:
            ip1, ids1, _ = gen.make_shard(cfg, 0, n_sets, dev, n_sets)
            want = signatures_csr(ip1, ids1, fam, out_dtype="uint32").cpu()
            q.put(("ok", bool(torch.equal(full.view(torch.int32), want.view(torch.int32))), cuts))
    except Exception as exc:
        q.put(("error", repr(exc), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_name,n_sets", [(2, "cfg2", 30_000), (3, "cfg3", 20_000), (2, "cfg5", 40_000)])
def test_split_gather_equals_single_process(cuda_device, world, cfg_name, n_sets):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_shard_worker, args=(world, _free_port(), cfg_name, n_sets, q), nprocs=world, join=True,
                       start_method="spawn")
    status, equal, cuts = q.get(timeout=60)
    assert status == "ok", equal
    assert equal, f"gathered shards differ from the single-process batch (cuts {cuts})"


def _nccl_worker(rank, world, port, q):
    """The NCCL backend itself (one rank: the box has one GPU): process-group init with a
    device id, the device-side cuts, sign_sharded's collective error agreement and the
    unpadded gather, and sign_gather_peer -- the same calls the multi-GPU bench makes."""
    import torch
    import torch.distributed as dist

    from paper_1401_6124_b200 import gen, make_family, signatures_csr
    from paper_1401_6124_b200.dist import nnz_balanced_cuts, sign_gather_peer, sign_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        cfg = gen.CONFIGS["cfg2"]
        ip_g = gen.global_indptr(cfg, dev, 20_000)
        ip, ids, _ = gen.make_shard(cfg, 0, 20_000, dev, 20_000, indptr=ip_g)
        assert nnz_balanced_cuts(ip, 1) == [0, 20_000]
        fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
        want = signatures_csr(ip, ids, fam, out_dtype="uint32")
        block, (s0, s1), full = sign_sharded(ip, ids, fam)
        ok = bool(torch.equal(full.view(torch.int32), want.view(torch.int32))) and (s0, s1) == (0, 20_000)
        mat, _ = sign_gather_peer(ip, ids, fam)
        ok = ok and bool(torch.equal(mat.tensor().view(torch.int32), want.view(torch.int32)))
        mat.close()
        bad_ids = ids.clone()
        bad_ids[5] = cfg.prime  # an id >= p: the reference's ValueError, agreed over the group
        try:
            sign_sharded(ip, bad_ids, fam)
            ok = False
        except ValueError:
            pass
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        dist.barrier()
        q.put(("ok", ok and float(t.item()) == 1.0))
    except Exception as exc:
        q.put(("error", repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def test_nccl_backend_one_rank(cuda_device):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_nccl_worker, args=(1, _free_port(), q), nprocs=1, join=True, start_method="spawn")
    status, ok = q.get(timeout=60)
    assert status == "ok" and ok, ok
