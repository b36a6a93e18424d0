"""Prime selection and modular helpers (host side).

Mirrors the reference's ``minhashlab.modmath`` API (modmath.py:1-65): the
same names, the same deterministic Miller-Rabin witness set, the same
``next_prime`` contract, and the same ``MAX_VECTOR_PRIME`` constant.  These
run once per family, never per visit.
"""
from __future__ import annotations

# Witnesses that make Miller-Rabin deterministic below 3.3e24 (reference modmath.py:11-13).
_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)

PRIME_SEARCH_LIMIT = 2**63 - 1          # reference modmath.py:17
MAX_VECTOR_PRIME = 3_037_000_499        # reference modmath.py:19: P*P + P < 2**63

# Largest modulus the u32 CUDA kernels accept (all residues and 2p fit in 32 bits).
MAX_KERNEL_PRIME = 2**31 - 1


def mulmod(a: int, x: int, p: int) -> int:
    """(a * x) % p with Python's unbounded ints (reference modmath.py:22-24)."""
    return (a * x) % p


def is_prime(n: int) -> bool:
    """Deterministic primality for 64-bit n (same decisions as modmath.py:27-47)."""
    if n < 2:
        return False
    for w in _WITNESSES:
        if n % w == 0:
            return n == w
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for w in _WITNESSES:
        y = pow(w, d, n)
        if y in (1, n - 1):
            continue
        for _ in range(r - 1):
            y = y * y % n
            if y == n - 1:
                break
        else:
            return False
    return True


def next_prime(n: int) -> int:
    """Smallest prime >= n; ValueError for n < 2, OverflowError past 2^63-1
    (reference modmath.py:50-65)."""
    if n < 2:
        raise ValueError(f"next_prime needs n >= 2, got {n}")
    if n == 2:
        return 2
    c = n if n % 2 else n + 1
    while c <= PRIME_SEARCH_LIMIT:
        if is_prime(c):
            return c
        c += 2
    raise OverflowError(f"no prime at or above {n} within the 64-bit search range")


def choose_prime(max_id: int, hashes: int, requested: int | None = None) -> int:
    """Smallest usable modulus (reference bench.py:66-70): above every feature id,
    with headroom for an iterative family of `hashes` members, honouring a floor."""
    return next_prime(max(max_id + 1, 2 * hashes + 3, requested or 0, 2))


def inv_mod(w: int, p: int) -> int:
    """w^{-1} mod prime p."""
    return pow(int(w) % p, -1, p)
