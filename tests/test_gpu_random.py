"""Randomised GPU parity: many small random CSR batches against the CPU oracle.

Each case draws a prime (small, BASELINE-sized, near the 3p < 2^32 boundary, or
wide >= 2^31), a family kind and size N, a set-size mix (singletons, sizes around
the 1024-feature chunk, long sets), unsorted rows with repeats, and an output
dtype.  Bar: bit-exact.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import make_family, next_prime, signatures_csr

pytestmark = pytest.mark.gpu

PRIMES = [11, 101, 7757, 65_537, 1_048_583, 16_777_259, 1_431_655_777, 2_147_483_647, 2_147_483_659,
          4_294_967_311]


def _case(seed):
    rng = np.random.default_rng(seed)
    p = int(rng.choice(PRIMES))
    if rng.random() < 0.3:
        p = next_prime(int(rng.integers(3, 1 << 31)))
    kind = ("random", "iterative")[int(rng.integers(0, 2))]
    n_max = max(1, min(3000, (p - 3) // 2))
    n = int(rng.choice([1, 2, 5, 16, 31, 64, 128, 200, 256, 511, 1000, 2048, 3000]))
    n = min(n, n_max)
    n_sets = int(rng.integers(1, 120))
    sizes = rng.choice([1, 2, 3, 50, 1023, 1024, 1025, 2500], size=n_sets,
                       p=[.1, .1, .1, .55, .03, .04, .03, .05])
    id_space = min(p, 1 << 32)
    rows = []
    for k in sizes:
        k = int(min(k, id_space))
        r = rng.integers(0, id_space, size=k, dtype=np.int64)
        if rng.random() < 0.3:  # repeats
            r = np.concatenate([r, r[: max(1, k // 3)]])
        rows.append(rng.permutation(r))
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    ids = np.concatenate(rows).astype(np.int64)
    fam = make_family(kind, int(rng.integers(0, 2**62)), n, p)
    dt = ("uint32", "int64")[int(rng.integers(0, 2))]
    return indptr, ids, fam, dt


@pytest.mark.parametrize("seed", range(40))
def test_random_batches_vs_oracle(cuda_device, seed):
    import torch

    indptr, ids, fam, dt = _case(seed)
    ip = torch.as_tensor(indptr, device=cuda_device)
    di = torch.as_tensor(ids, device=cuda_device)
    got = signatures_csr(ip, di, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
    if fam.prime <= 3_037_000_499:
        want = oracle.sign_family_csr(indptr, ids.astype(np.uint32), fam)
    else:  # beyond the int64 oracle: Python-int brute force per row
        want = np.stack([oracle.brute_force_row(ids[indptr[s]:indptr[s + 1]], fam) for s in range(indptr.size - 1)])
    assert np.array_equal(got, want), (fam, dt)
