"""GPU parity of the output-sensitive iterative kernel (csrc/gap.cu) against the CPU oracle.

The kernel enumerates, per feature, only the hash lanes whose value falls under the
set's threshold (three-gap structure of the iterative family's arithmetic progression,
kernels.py:62-72) and recomputes the rare entries that stay above it.  ``MHB_GAP=1``
forces it for every batch above the small-batch plan (16,384 sets); the cases below
cover the descent's corners: tiny and huge sets (thresholds p and 1), repeats, the
constant orbit x = p - b, primes from 101 to 2^31 - 1, lane counts that are not a
multiple of four or exceed the register-resident tables, both output dtypes, and the
status flags.  Bar: bit-exact.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import make_family, signatures_csr

pytestmark = pytest.mark.gpu

N_SETS = 16_500  # just above the small-batch plan, so the sorted plan's hook is taken


@pytest.fixture(autouse=True)
def _force_gap(monkeypatch):
    monkeypatch.setenv("MHB_GAP", "1")


def _batch(rng, p, sizes, id_space=None):
    id_space = min(p, 1 << 32) if id_space is None else id_space
    rows = []
    for k in sizes:
        r = rng.integers(0, id_space, size=int(k), dtype=np.int64)
        if rng.random() < 0.2:
            r = np.concatenate([r, r[: max(1, int(k) // 3)]])
        rows.append(r)
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return indptr, np.concatenate(rows).astype(np.int64)


def _check(cuda_device, indptr, ids, fam, dt="uint32", rows=None):
    import torch

    ip = torch.as_tensor(indptr, device=cuda_device)
    di = torch.as_tensor(ids, device=cuda_device)
    got = signatures_csr(ip, di, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
    sel = np.arange(indptr.size - 1) if rows is None else rows
    for s0 in range(0, sel.size, 4096):
        part = sel[s0:s0 + 4096]
        sub_ip = np.concatenate([[0], np.cumsum(indptr[part + 1] - indptr[part])]).astype(np.int64)
        sub_ids = np.concatenate([ids[indptr[s]:indptr[s + 1]] for s in part]).astype(np.uint32)
        want = oracle.sign_family_csr(sub_ip, sub_ids, fam)
        assert np.array_equal(got[part], want), (fam.prime, fam.size, dt)


@pytest.mark.parametrize("p,n_hash,dt", [
    (67_108_879, 2048, "uint32"),      # cfg4's prime and lane count
    (67_108_879, 130, "int64"),        # not a multiple of four: scalar row path
    (4_194_319, 512, "uint32"),        # cfg3
    (16_777_259, 256, "int64"),        # cfg2
    (1_073_741_827, 256, "uint32"),    # cfg5: 3p >= 2^32
    (2_147_483_647, 1000, "uint32"),   # largest 31-bit prime
    (67_108_879, 2500, "uint32"),      # lane tables read from memory (N > 2048)
    (7757, 64, "int64"),
])
def test_gap_kernel_vs_oracle(cuda_device, p, n_hash, dt):
    rng = np.random.default_rng(p % 1000 + n_hash)
    sizes = rng.choice([1, 2, 3, 17, 80, 300, 1500], size=N_SETS, p=[.05, .05, .05, .25, .5, .09, .01])
    indptr, ids = _batch(rng, p, sizes)
    fam = make_family("iterative", int(rng.integers(0, 2**62)), n_hash, p)
    rows = np.unique(np.concatenate([np.arange(300), rng.integers(0, N_SETS, 900), np.flatnonzero(sizes >= 300)[:40]]))
    _check(cuda_device, indptr, ids, fam, dt, rows)


def test_gap_small_prime_thresholds_of_one(cuda_device):
    """p = 101 with sets of up to 3,000 (repeated) ids: the threshold p c / n bottoms out
    at 1, the descent runs to its last level, and most lanes' minimum is 0."""
    rng = np.random.default_rng(5)
    p = 101
    sizes = rng.choice([1, 5, 40, 700, 3000], size=N_SETS, p=[.2, .3, .3, .15, .05])
    indptr, ids = _batch(rng, p, sizes)
    fam = make_family("iterative", 11, 40, p)
    _check(cuda_device, indptr, ids, fam, "uint32", np.arange(0, N_SETS, 7))


def test_gap_constant_orbit_and_extremes(cuda_device):
    """x = p - b makes d = (x + b) mod p = 0: every lane hashes x to the same value.  Also
    ids 0 and p - 1, and one 20,000-id set in a tile of singletons."""
    rng = np.random.default_rng(9)
    p = 16_777_259
    fam = make_family("iterative", 3, 256, p)
    x0 = (p - fam.base.b) % p
    rows = []
    for s in range(N_SETS):
        k = s % 5
        if k == 0:
            rows.append(np.array([x0], dtype=np.int64))
        elif k == 1:
            rows.append(np.array([x0, 0, p - 1], dtype=np.int64))
        elif k == 2:
            rows.append(np.concatenate([[x0], rng.integers(0, p, 60)]).astype(np.int64))
        elif k == 3:
            rows.append(np.array([p - 1], dtype=np.int64))
        else:
            rows.append(rng.integers(0, p, 90).astype(np.int64))
    rows[1234] = rng.integers(0, p, 20_000).astype(np.int64)
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    ids = np.concatenate(rows)
    sel = np.unique(np.concatenate([np.arange(400), np.arange(1200, 1270)]))
    _check(cuda_device, indptr, ids, fam, "int64", sel)


def test_gap_sets_of_one_repeated_id(cuda_device):
    """Sets of thousands of copies of one id: the threshold (sized for n distinct features)
    is far too low, nearly every lane goes to the fallback, the result is still exact."""
    rng = np.random.default_rng(13)
    p = 67_108_879
    fam = make_family("iterative", 9, 512, p)
    rows = [rng.integers(0, p, 70).astype(np.int64) for _ in range(N_SETS)]
    for s in (5, 4000, 16_499):
        rows[s] = np.full(6000, int(rng.integers(0, p)), dtype=np.int64)
    rows[77] = np.concatenate([np.full(3000, 12345), np.full(3000, 54321)]).astype(np.int64)
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    sel = np.unique(np.concatenate([np.arange(0, 120), np.arange(3990, 4010), np.arange(16_490, 16_500)]))
    _check(cuda_device, indptr, np.concatenate(rows), fam, "uint32", sel)


def test_gap_matches_visiting_kernel_everywhere(cuda_device, monkeypatch):
    """The whole matrix of a cfg4-shaped batch equals the visiting kernel's, entry by entry."""
    import torch

    from paper_1401_6124_b200 import gen

    cfg = gen.CONFIGS["cfg4"]
    indptr, ids = gen.make_csr(cfg, cuda_device, n_sets=60_000)
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    got = signatures_csr(indptr, ids, fam, out_dtype="uint32")
    monkeypatch.setenv("MHB_GAP", "0")
    want = signatures_csr(indptr, ids, fam, out_dtype="uint32")
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))


def test_gap_fallback_list_overflow(cuda_device, monkeypatch):
    """A threshold scale of 1e-4 drops c to its floor of 1: ~37% of the entries stay above
    the threshold, far more than the tile's fallback list holds, so the marked-minima
    pass redoes them in place."""
    monkeypatch.setenv("MHB_GAP_CMUL", "0.0001")
    rng = np.random.default_rng(21)
    p = 67_108_879
    indptr, ids = _batch(rng, p, rng.choice([40, 80, 120], size=N_SETS))
    for n_hash, dt in ((2048, "uint32"), (250, "int64")):
        fam = make_family("iterative", 77, n_hash, p)
        _check(cuda_device, indptr, ids, fam, dt, np.arange(0, N_SETS, 41))


def test_gap_small_batches_with_a_full_wave(cuda_device, monkeypatch):
    """Batches the small-batch plan could take go to the enumerating kernel once they make
    a full wave of tiles (cfg4 shape: 3,552 sets); MHB_GAP_MIN_SETS moves the floor."""
    rng = np.random.default_rng(17)
    p = 67_108_879
    fam = make_family("iterative", 31, 2048, p)
    for n_sets, floor_sets in ((4000, None), (700, "1"), (37, "1")):
        if floor_sets is None:
            monkeypatch.delenv("MHB_GAP_MIN_SETS", raising=False)
        else:
            monkeypatch.setenv("MHB_GAP_MIN_SETS", floor_sets)
        indptr, ids = _batch(rng, p, np.maximum(1, rng.poisson(80, size=n_sets)))
        _check(cuda_device, indptr, ids, fam, "uint32", np.arange(0, n_sets, max(1, n_sets // 150)))


def test_gap_status_flags(cuda_device):
    import torch

    rng = np.random.default_rng(3)
    p = 1_048_583
    fam = make_family("iterative", 5, 128, p)
    indptr, ids = _batch(rng, p, np.full(N_SETS, 20))
    bad = ids.copy()
    bad[777] = p + 5
    with pytest.raises(ValueError, match="prime"):
        signatures_csr(torch.as_tensor(indptr, device=cuda_device),
                       torch.as_tensor(bad, device=cuda_device).to(torch.uint32), fam)
    ip2 = indptr.copy()
    ip2[501:] -= 20  # set 500 becomes empty
    with pytest.raises(ValueError, match="empty"):
        signatures_csr(torch.as_tensor(ip2, device=cuda_device),
                       torch.as_tensor(ids[:-20], device=cuda_device).to(torch.uint32), fam)
