"""ctypes binding of libmhb.so (the C ABI declared in include/mhb.h).

The library is the product path: there is no CPU fallback.  If the shared
object is missing or fails to load, every GPU entry point raises
``NativeLibraryError`` instead of computing anything another way.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

# MHB_LIB overrides the library path (A/B experiments with variant builds).
LIB_PATH = Path(os.environ.get("MHB_LIB") or Path(__file__).resolve().parent / "lib" / "libmhb.so")

MHB_OK = 0
MHB_ERR_INVALID = 1
MHB_ERR_CUDA = 2
MHB_ERR_UNSUPPORTED = 3

OUT_U32 = 0
OUT_I64 = 1

STATUS_EMPTY_SET = 1
STATUS_ID_GE_PRIME = 2
STATUS_BAD_PARAM = 4

KIND_ITERATIVE = 0
KIND_RANDOM = 1

# Every symbol include/mhb.h declares, with (restype, argtypes).
_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_I32 = C.c_int32
_U32 = C.c_uint32
_SZ = C.c_size_t
SIGNATURES = {
    "mhb_version": (C.c_char_p, []),
    "mhb_last_error": (C.c_char_p, []),
    "mhb_sign_workspace_bytes": (_SZ, [_I64, _I64, _I32]),
    "mhb_sign_iterative_path": (_I32, [_I64, _I64, _U64, _I32]),
    "mhb_sign_iterative_csr": (C.c_int, [_P, _P, _I64, _I64, _U64, _U64, _U64, _I32, _P, _I32, _P, _P, _SZ, _P]),
    "mhb_sign_random_csr": (C.c_int, [_P, _P, _I64, _I64, _P, _P, _U64, _I32, _P, _I32, _P, _P, _SZ, _P]),
    "mhb_sign_iterative_csr_bands": (C.c_int, [_P, _P, _I64, _I64, _U64, _U64, _U64, _I32, _I32, _P, _P, _I32,
                                               _I32, _P, _P, _SZ, _P]),
    "mhb_sign_random_csr_u64": (C.c_int, [_P, _P, _I64, _I64, _P, _P, _U64, _I32, _P, _I32, _P, _P]),
    "mhb_sign_csr_ids64": (C.c_int, [_I32, _P, _P, _I64, _I64, _U64, _U64, _P, _P, _U64, _I32, _P, _P, _P]),
    "mhb_sign_csr_host": (C.c_int, [_I32, _P, _P, _I64, _I64, _U64, _U64, _P, _P, _U64, _I32, _P, _I32, _P, _I32]),
    "mhb_host_release": (None, []),
    "mhb_host_pool_selftest": (C.c_int, [_I64, _U64, _I32, _P]),
    "mhb_jaccard_pairs": (C.c_int, [_P, _I32, _I32, _P, _P, _I64, _P, _P, _P]),
    "mhb_jaccard_block": (C.c_int, [_P, _I64, _P, _I64, _I32, _I32, _P, _P]),
    "mhb_band_keys": (C.c_int, [_P, _I32, _I64, _I32, _I32, _P, _P]),
    "mhb_format_binary_records": (C.c_int, [_P, _I32, _I64, _I32, _P, _I64, _P, _P]),
    "mhb_text_record_lengths": (C.c_int, [_P, _I32, _I64, _I32, _P, _I64, _P, _P]),
    "mhb_format_text_records": (C.c_int, [_P, _I32, _I64, _I32, _P, _I64, _P, _P, _P]),
    "mhb_bucket_hist_iterative": (C.c_int, [_P, _I64, _U64, _U64, _U64, _I32, _U32, _P, _P]),
    "mhb_bucket_hist_random": (C.c_int, [_P, _I64, _P, _P, _U64, _I32, _U32, _P, _P]),
    "mhb_bucket_hist_u64": (C.c_int, [_I32, _P, _I64, _U64, _U64, _P, _P, _U64, _I32, _U64, _P, _P]),
    "mhb_corpus_scan": (C.c_int, [_P, _I64, _I32, _P]),
    "mhb_corpus_scan_device": (C.c_int, [_P, _I64, _I32, _P, _P]),
    "mhb_corpus_info": (C.c_int, [_P, _P, _P]),
    "mhb_corpus_deferred": (C.c_int, [_P, _P, _P, _P]),
    "mhb_corpus_set_terms": (C.c_int, [_P, _I64, _P, _P, _P, _P]),
    "mhb_corpus_intern": (C.c_int, [_P, _P, _P, _P, _P]),
    "mhb_corpus_export": (C.c_int, [_P, _P, _P, _P, _P]),
    "mhb_corpus_export_device": (C.c_int, [_P, _P, _P, _P]),
    "mhb_corpus_free": (None, [_P]),
    "mhb_peer_alloc": (C.c_int, [_SZ, _I32, _P, _P]),
    "mhb_peer_open": (C.c_int, [_P, _I32, _P]),
    "mhb_peer_close": (C.c_int, [_P]),
    "mhb_peer_free": (C.c_int, [_P]),
    "mhb_probe_visit_rate": (C.c_int, [_I64, _I32, C.POINTER(C.c_double), C.POINTER(C.c_float), _P]),
    "mhb_profile_begin": (C.c_int, [_I32]),
    "mhb_profile_end": (C.c_int, [C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
}


class NativeLibraryError(RuntimeError):
    """libmhb.so is missing or unusable; there is deliberately no fallback."""


class MhbError(RuntimeError):
    """A libmhb call returned an error code."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libmhb error {code}: {message}")
        self.code = code
        self.message = message


_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load (once) and return the ctypes handle, with every prototype declared."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load().mhb_last_error().decode()


def check(code: int) -> None:
    """Raise the reference's exception type for argument errors, MhbError otherwise."""
    if code == MHB_OK:
        return
    msg = last_error()
    if code == MHB_ERR_INVALID:
        raise ValueError(msg)
    if code == MHB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise MhbError(code, msg)
