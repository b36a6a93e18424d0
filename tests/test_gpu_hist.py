"""Bucket-uniformity histogram kernels (aux.cu) against the oracle's restatement of
stats.py:221-224 (bincount(eval_all(x) % m) summed over a batch of x).

Covers both kernels the library routes between -- the per-lane byte-replica kernel
(m <= 4096, power of two or not) and the u32 table fallback (m > 4096) -- the 64-bit
kernel for primes >= 2^31, and the byte counters' 127 -> 128 spill: inputs whose
iterative step dh is a multiple of 4096 keep hundreds of consecutive members in ONE
bin, far past what a byte holds."""
import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import bucket_histogram, make_family

pytestmark = pytest.mark.gpu


def _np_hist_iter(fam, xs, m):
    """Vectorised restatement for p < 2^31 (int64 exact): h_i(x) = (a x + i ((x+b) mod p)) mod p."""
    p, a, b = fam.prime, fam.base.a, fam.base.b
    xs = np.asarray(xs, dtype=np.int64)
    counts = np.zeros(m, dtype=np.int64)
    h = (a * xs) % p
    d = (xs + b) % p
    for _ in range(fam.size):
        counts += np.bincount(h % m, minlength=m)
        h = (h + d) % p
    return counts


@pytest.mark.parametrize("m", [1, 2, 3, 4, 64, 100, 4095, 4096, 5000, 70000])
@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_hist_bucket_counts(cuda_device, m, kind):
    rng = np.random.default_rng(m)
    p = 4_194_319
    fam = make_family(kind, 11, 96, p)
    xs = rng.choice(p, size=300, replace=False)
    got = bucket_histogram(xs, fam, m).cpu().numpy()
    assert got.tolist() == oracle.bucket_histogram(fam, xs, m).tolist()


@pytest.mark.parametrize("n_hash", [1, 5, 63, 64, 65, 512, 2048, 3000])
def test_hist_member_counts(cuda_device, n_hash):
    p = 67_108_879  # cfg4's prime (3p >= 2^32 for none; >= 2^24)
    fam = make_family("iterative", 3, n_hash, p)
    xs = np.random.default_rng(n_hash).choice(p, size=500, replace=False)
    got = bucket_histogram(xs, fam, 4096).cpu().numpy()
    assert got.tolist() == _np_hist_iter(fam, xs, 4096).tolist()
    famr = make_family("random", 3, n_hash, 16_777_259)
    xs = xs % 16_777_259
    xs = np.unique(xs)
    assert bucket_histogram(xs, famr, 4096).cpu().numpy().tolist() == oracle.bucket_histogram(famr, xs, 4096).tolist()


def test_hist_byte_spill(cuda_device):
    """dh = (x + b) mod p a multiple of 4096 and far below p: a whole run of members
    shares one bin (thousands of increments of one byte counter per thread)."""
    p = 1_073_741_827  # cfg5's prime
    fam = make_family("iterative", 5, 2048, p)
    b = fam.base.b
    t = np.arange(1, 4001, dtype=np.int64)
    xs = np.unique((4096 * t - b) % p)
    got = bucket_histogram(xs, fam, 4096).cpu().numpy()
    want = _np_hist_iter(fam, xs, 4096)
    assert want.max() >= 2048  # the case really concentrates (a whole x in one bin)
    assert got.tolist() == want.tolist()


def test_hist_large_batch_vs_vectorised(cuda_device):
    """A cfg3-shaped run: many x (every one of 2^18 ids) x 512 members into 64x64 bins."""
    p = 4_194_319
    fam = make_family("iterative", 9, 512, p)
    xs = np.arange(1 << 18, dtype=np.int64)
    got = bucket_histogram(xs, fam, 4096).cpu().numpy()
    assert got.tolist() == _np_hist_iter(fam, xs, 4096).tolist()
    assert int(got.sum()) == xs.size * 512


@pytest.mark.parametrize("kind", ["iterative", "random"])
@pytest.mark.parametrize("p", [2_147_483_659, 4_294_967_311, (1 << 61) - 1])
def test_hist_wide_primes(cuda_device, kind, p):
    """Primes >= 2^31 (the reference counts for any prime, families.py:105-112)."""
    fam = make_family(kind, 2, 40, p)
    rng = np.random.default_rng(1)
    xs = np.unique(rng.integers(0, min(p, 1 << 62), size=200, dtype=np.int64))
    for m in (4096, 7, 1):
        got = bucket_histogram(xs, fam, m).cpu().numpy()
        assert got.tolist() == oracle.bucket_histogram(fam, xs, m).tolist(), m


def test_hist_rejects_out_of_range(cuda_device):
    fam = make_family("iterative", 2, 8, 1_048_583)
    with pytest.raises(ValueError):
        bucket_histogram([0, 1_048_583], fam, 16)
    with pytest.raises(ValueError):
        bucket_histogram([1], fam, 0)
