"""The C ABI library loads, exports every symbol include/mhb.h declares, and
rejects bad arguments before touching CUDA (CPU only, no kernel launches)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1401_6124_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "mhb.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mhb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for name in ("mhb_sign_iterative_csr", "mhb_sign_random_csr", "mhb_sign_csr_host", "mhb_jaccard_pairs",
                 "mhb_bucket_hist_iterative", "mhb_last_error", "mhb_sign_workspace_bytes"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version_and_error_text():
    lib = _lib.load()
    assert b"sm_100a" in lib.mhb_version()
    assert isinstance(_lib.last_error(), str)


def test_workspace_bytes_monotone():
    lib = _lib.load()
    a = lib.mhb_sign_workspace_bytes(1000, 50_000, 256)
    b = lib.mhb_sign_workspace_bytes(1000, 5_000_000, 256)
    c = lib.mhb_sign_workspace_bytes(1000, 50_000, 4096)
    assert 0 < a < b and a < c


@pytest.mark.parametrize("prime,a,n,err", [
    (7758, 1, 4, "not prime"),            # non-prime modulus (families.py:46-50)
    (7757, 7755, 4, "a + size < prime"),   # headroom (families.py:140-145)
    (7757, 0, 4, "1 <= a < p"),
])
def test_argument_errors_before_launch(prime, a, n, err):
    lib = _lib.load()
    rc = lib.mhb_sign_iterative_csr(None, None, 0, 0, a, 3, prime, n, None, 0, None, None, 0, None)
    assert rc == _lib.MHB_ERR_INVALID
    assert err in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_prime_range_limits():
    lib = _lib.load()
    p63 = 2**63 + 29  # first prime above 2^63: beyond the reference's 64-bit range too
    rc = lib.mhb_sign_iterative_csr(None, None, 0, 0, 5, 3, p63, 4, None, 0, None, None, 0, None)
    assert rc == _lib.MHB_ERR_UNSUPPORTED
    with pytest.raises(NotImplementedError):
        _lib.check(rc)
    wide = 2_147_483_659  # smallest prime above 2^31: supported (64-bit path), no work for n_sets=0
    assert lib.mhb_sign_iterative_csr(None, None, 0, 0, 5, 3, wide, 4, None, 0, None, None, 0, None) == _lib.MHB_OK
    dummy = C.c_int64(0)
    rc = lib.mhb_sign_random_csr(None, None, 0, 0, C.addressof(dummy), C.addressof(dummy), wide, 4,
                                 None, 0, None, None, 0, None)
    assert rc == _lib.MHB_ERR_UNSUPPORTED and "u64" in _lib.last_error()


def test_workspace_too_small_rejected():
    lib = _lib.load()
    dummy = C.c_int64(0)
    rc = lib.mhb_sign_iterative_csr(C.addressof(dummy), C.addressof(dummy), 1, 1, 5, 3, 7757, 4,
                                    C.addressof(dummy), 0, None, C.addressof(dummy), 8, None)
    assert rc == _lib.MHB_ERR_INVALID and "workspace" in _lib.last_error()


def test_workspace_bytes_fit_smaller_batches():
    """A workspace sized for a batch fits every smaller batch: the virtual-set size
    shrinks with the batch (choose_chunk), so the bound must not (host-only call)."""
    from paper_1401_6124_b200 import _lib

    lib = _lib.load()
    for n_hash in (1, 128, 256, 2048, 100_000):
        for n_sets in (1, 1000, 1_000_000):
            prev = 0
            for nnz in [0, 10, 10**4] + [int(1e5 * 1.25**k) for k in range(60)]:
                b = lib.mhb_sign_workspace_bytes(n_sets, nnz, n_hash)
                assert b >= prev, (n_hash, n_sets, nnz)
                prev = b
