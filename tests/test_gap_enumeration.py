"""CPU pin of the enumeration the iterative family's output-sensitive kernel runs
(csrc/gap.cu `enumerate_feature`), restated in Python integers and checked against
brute force: for h_i = (h0 + i d) mod p (kernels.py:62-72: lane i of the iterative family
hashes x to h_0(x) + i (x + b)), list every i < N with h_i < T.

The restatement follows the CUDA line by line (one level of the descent with both cases
in one stream, the carried entry point, the return map as an upward step and a downward
step under two predicates), so a change to the kernel's arithmetic has a CPU counterpart to update.
Also here: the cost model's choices for the BASELINE shapes through the C ABI
(`mhb_sign_iterative_path`, host logic only -- no GPU call).
"""
import random

import pytest

from paper_1401_6124_b200 import _lib, gen


def enumerate_hits(p, d, h0, T, N):
    """[(i, h_i)] for every i < N with h_i < T, in increasing i -- gap.cu's walk."""
    v, t = h0, 0
    if d == 0:
        if v >= T:
            return []
        u, n, w, m = 0, 1, T, N
    else:
        u, n, w, m = d, 1, p - d, 1
        L = p
        while True:
            mn = min(u, w)
            if mn == 0 or L - mn < T or t >= N:
                break
            up_big = u >= w
            big, tb, ts = (u, n, m) if up_big else (w, m, n)
            j = min(big, L - T) // mn
            L2 = L - j * mn
            if v >= L2:
                q = ((v - L2) if up_big else (L - 1 - v)) // mn
                v -= (q + 1) * mn if up_big else big - q * mn
                t += (q + 1) * ts if up_big else tb + q * ts
            big2, tb2 = big - j * mn, tb + j * ts
            if up_big:
                u, n = big2, tb2
            else:
                w, m = big2, tb2
            L = L2
        if t >= N:
            return []
        if v >= T:
            v -= w
            t += m
            if t >= N:
                return []
    out = []
    while t < N:
        out.append((t, v))
        up = v < w
        if up:
            v += u
            t += n
        if not (up and v < T):  # no upward step, or one that overshot T: the downward step
            v -= w
            t += m
    return out


@pytest.mark.parametrize("seed", range(8))
def test_enumeration_matches_brute_force(seed):
    rng = random.Random(seed)
    primes = [7, 13, 101, 7757, 1_048_583, 4_194_319, 16_777_259, 67_108_879, 1_073_741_827, 2_147_483_647]
    for _ in range(1500):
        p = rng.choice(primes)
        d = rng.choice([0, 1, p - 1, 2, p // 2]) if rng.random() < 0.1 else rng.randrange(0, p)
        d %= p
        h0 = rng.randrange(0, p)
        T = rng.choice([1, 2, max(1, p // 20), max(1, p // 300), p, p - 1, max(1, p // 2), rng.randrange(1, p + 1)])
        N = min(rng.choice([1, 2, 128, 256, 2048]), p - 1)
        got = enumerate_hits(p, d, h0, T, N)
        want = [(i, (h0 + i * d) % p) for i in range(N) if (h0 + i * d) % p < T]
        assert got == want, (p, d, h0, T, N)


def test_cost_model_choices_for_baseline_shapes(monkeypatch):
    """cfg4 and cfg3 (many lanes per feature) take the enumerating kernel; cfg2 / cfg5
    (N = 256) and small batches short of a full wave of tiles keep the visiting kernel; MHB_GAP forces."""
    monkeypatch.delenv("MHB_GAP", raising=False)
    lib = _lib.load()

    def path(name, n_sets, mean):
        cfg = gen.CONFIGS[name]
        return lib.mhb_sign_iterative_path(n_sets, int(n_sets * mean), cfg.prime, cfg.n_hash)

    assert path("cfg4", 2_000_000, 80) == 1
    assert path("cfg4", 250_000, 80) == 1          # an 8-GPU shard
    assert path("cfg3", 400_000, 300) == 1
    assert path("cfg2", 1_000_000, 198) == 0
    assert path("cfg5", 12_500_000, 123) == 0
    assert path("cfg1", 10_000, 50) == 0
    assert path("cfg4", 16_384, 80) == 1           # a full wave of tiles (592 x 6 sets) and more
    assert path("cfg4", 3_000, 80) == 0            # under a wave: the small-batch plan
    assert path("cfg3", 8_000, 300) == 0           # 24-set tiles: a wave is 14,208 sets
    monkeypatch.setenv("MHB_GAP", "0")
    assert path("cfg4", 2_000_000, 80) == 0
    monkeypatch.setenv("MHB_GAP", "1")
    assert path("cfg2", 1_000_000, 198) == 1
    assert path("cfg4", 3_000, 80) == 0            # still the small-batch plan
    assert lib.mhb_sign_iterative_path(100_000, 8_000_000, 2**31 + 11, 256) == 0   # wide primes: wide.cu
