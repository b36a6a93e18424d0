"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the MinHash signature path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline -- never as the thing measured or shipped.  The product
(``paper_1401_6124_b200``) does not import it and has no CPU fallback.

Contents
  * ctypes loader for ``minhash_oracle.c`` -- the C restatement of the
    reference's numba loops (kernels.py:21-73), OpenMP across rows.
  * numpy restatements of the other parity targets:
      bucket histogram   stats.py:221-224   bincount(eval_all(x) % buckets)
      Jaccard estimate   minhash.py:130-137 mean(g1 == g2)
      brute force        tests/test_minhash.py:27-39 (per-hash scan with eval_at)

Pinning: tests/test_oracle.py checks this oracle against every known-answer
vector of the reference tests and against golden outputs produced by running
the reference itself (tests/golden/make_golden.py, committed fixtures).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "minhash_oracle.c"
LIB = HERE / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    """gcc -O2 -fopenmp the C restatement into oracle/liboracle.so."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        cmd = ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", str(SRC), "-o", str(LIB)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"oracle build failed: {r.stderr}")
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(LIB))
        P, I64, I32 = C.c_void_p, C.c_int64, C.c_int32
        lib.oracle_sign_iterative_csr.argtypes = [P, P, I64, I64, I64, I64, I32, P, I32]
        lib.oracle_sign_iterative_csr.restype = None
        lib.oracle_sign_random_csr.argtypes = [P, P, I64, P, P, I64, I32, P, I32]
        lib.oracle_sign_random_csr.restype = None
        lib.oracle_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(load().oracle_max_threads())


def _csr(indptr, ids):
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    return indptr, ids


def sign_iterative_csr(indptr, ids, a: int, b: int, p: int, n: int, threads: int = 0) -> np.ndarray:
    """int64[S, n] argmin ids, reference kernels.sign_iterative applied per row."""
    indptr, ids = _csr(indptr, ids)
    s = indptr.size - 1
    out = np.zeros((s, n), dtype=np.int64)
    load().oracle_sign_iterative_csr(indptr.ctypes.data, ids.ctypes.data, s, int(a), int(b), int(p), int(n),
                                     out.ctypes.data, int(threads))
    return out


def sign_random_csr(indptr, ids, a, b, p: int, threads: int = 0) -> np.ndarray:
    """int64[S, N] argmin ids, reference kernels.sign_random applied per row."""
    indptr, ids = _csr(indptr, ids)
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    s = indptr.size - 1
    out = np.zeros((s, a.size), dtype=np.int64)
    load().oracle_sign_random_csr(indptr.ctypes.data, ids.ctypes.data, s, a.ctypes.data, b.ctypes.data, int(p),
                                  int(a.size), out.ctypes.data, int(threads))
    return out


def sign_family_csr(indptr, ids, family, threads: int = 0) -> np.ndarray:
    """Dispatch on a family object exposing the reference's attributes."""
    if family.kind == "iterative":
        return sign_iterative_csr(indptr, ids, family.base.a, family.base.b, family.prime, family.size, threads)
    return sign_random_csr(indptr, ids, family.a, family.b, family.prime, threads)


# --- numpy restatements ------------------------------------------------------

def member_values(family, x: int) -> np.ndarray:
    """All N hash values of x (families.py:105-112 / 153-168), exact in Python ints."""
    p = family.prime
    if family.kind == "iterative":
        a, b = family.base.a, family.base.b
        i = np.arange(family.size, dtype=object)
        return np.array(((a * x) + i * ((x + b) % p)) % p, dtype=np.int64)
    return np.array([(int(ai) * x + int(bi)) % p for ai, bi in zip(family.a, family.b)], dtype=np.int64)


def bucket_histogram(family, xs, buckets: int) -> np.ndarray:
    """sum over x in xs of bincount(eval_all(x) % buckets) (stats.py:222-224)."""
    counts = np.zeros(buckets, dtype=np.int64)
    for x in np.asarray(xs).tolist():
        counts += np.bincount(member_values(family, int(x)) % buckets, minlength=buckets)
    return counts


def jaccard_estimate(m1: np.ndarray, m2: np.ndarray) -> float:
    """float(np.mean(g1.mins == g2.mins)) (minhash.py:137)."""
    return float(np.mean(np.asarray(m1) == np.asarray(m2)))


def band_keys(sig: np.ndarray, rows_per_band: int) -> np.ndarray:
    """LSH band keys as defined in include/mhb.h / csrc/bandhash.cuh: over the band's
    argmin ids (uint32, row order) h1 <- h1*0x9E3779B1 + x and h2 <- h2*0x85EBCA6B + x
    mod 2^32, seeded 0x811C9DC5 ^ band and 0xC2B2AE35 ^ (band*0x27D4EB2F); the key is
    splitmix64(h1 << 32 | h2)."""
    sig = np.asarray(sig).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    n_sets, n_hash = sig.shape
    nb = n_hash // rows_per_band
    m32 = np.uint64(0xFFFFFFFF)
    band = np.arange(nb, dtype=np.uint64)[None, :].repeat(n_sets, 0)
    with np.errstate(over="ignore"):
        h1 = np.uint64(0x811C9DC5) ^ band
        h2 = np.uint64(0xC2B2AE35) ^ ((band * np.uint64(0x27D4EB2F)) & m32)
        blocks = sig.reshape(n_sets, nb, rows_per_band)
        for j in range(rows_per_band):
            h1 = (h1 * np.uint64(0x9E3779B1) + blocks[:, :, j]) & m32
            h2 = (h2 * np.uint64(0x85EBCA6B) + blocks[:, :, j]) & m32
        z = (h1 << np.uint64(32)) | h2
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def brute_force_row(ids, family) -> np.ndarray:
    """Per hash index, scan ascending ids, strict '<' (tests/test_minhash.py:27-39)."""
    ids = sorted(set(int(v) for v in ids))
    out = np.empty(family.size, dtype=np.int64)
    p = family.prime
    for i in range(family.size):
        best, arg = None, None
        for x in ids:
            if family.kind == "iterative":
                hv = (family.base.a * x + i * ((x + family.base.b) % p)) % p
            else:
                hv = (int(family.a[i]) * x + int(family.b[i])) % p
            if best is None or hv < best:
                best, arg = hv, x
        out[i] = arg
    return out


if os.environ.get("MHB_ORACLE_BUILD_ON_IMPORT"):
    build()
