"""The host copy pool behind mhb_sign_csr_host (csrc/host.cu HostPool): 10^5
back-to-back jobs of random part counts and uneven part lengths, from 4 concurrent
callers, each part must run exactly once.  Round 1's pool could hand a stale part
index of the previous job to a slow worker (double execution, an early return while
a staging copy still ran); claims are now CAS-tagged with the job generation.
Needs no GPU: the pool is plain host threads."""
import ctypes as C


def test_host_pool_runs_every_part_exactly_once():
    from paper_1401_6124_b200 import _lib

    lib = _lib.load()
    for seed, threads in ((7, 4), (11, 1), (13, 8)):
        bad = C.c_int64(-1)
        _lib.check(lib.mhb_host_pool_selftest(100_000 if threads != 8 else 30_000, seed, threads, C.byref(bad)))
        assert bad.value == 0, (seed, threads, bad.value)


import numpy as np
import pytest


@pytest.mark.gpu
def test_host_pipeline_back_to_back_mixed(cuda_device):
    """Back-to-back mhb_sign_csr_host calls of mixed sizes, pageable and pinned buffers,
    uint32 and int64 outputs (the pool stages pageable ids in and widens / copies the
    outputs), every result equal to the device path on the same batch."""
    import torch

    from paper_1401_6124_b200 import gen, make_family, signatures_csr

    cfg = gen.CONFIGS["cfg2"]
    fam = make_family("iterative", 5, 64, cfg.prime)
    batches = []
    for k, n in enumerate((700, 3000, 12000, 40000, 90000)):
        ip, ids = gen.make_csr(cfg, device=cuda_device, n_sets=n, seed=100 + k)
        want = signatures_csr(ip, ids, fam, out_dtype="int64").cpu().numpy()
        ip_h, ids_h = ip.cpu().numpy(), ids.cpu().numpy().view(np.uint32)
        ids_pin = torch.empty(ids_h.size, dtype=torch.int32, pin_memory=True)
        ids_pin.copy_(torch.from_numpy(ids_h.view(np.int32)))
        batches.append((ip_h, ids_h, ids_pin.numpy().view(np.uint32), want))
    rng = np.random.default_rng(3)
    for call in range(300):
        ip_h, ids_h, ids_p, want = batches[int(rng.integers(len(batches)))]
        src = ids_p if rng.random() < 0.5 else ids_h
        dt = "int64" if rng.random() < 0.5 else "uint32"
        got = signatures_csr(ip_h, src, fam, out_dtype=dt)
        assert np.array_equal(got.astype(np.int64), want), (call, dt)
