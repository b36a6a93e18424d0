"""Corpus ingest -> CSR, and the reference's ``sign`` command on top of it.

Mirrors ``minhashlab.corpus`` (reference src/corpus.py:18-80): ``tokenize``,
``Vocabulary``, ``CorpusData``, ``build_corpus`` keep their names, arguments and
results.  The work runs in libmhb behind one ``mhb_corpus_*`` handle API with two
backends, chosen explicitly by the caller (no automatic dispatch, no fallback):

* device (csrc/corpus_gpu.cu, ``backend="gpu"``, the default; it raises when no GPU is
  visible): tokens, vocabulary
  and documents are computed on the GPU; non-ASCII lines too, with this Python's own
  ``str.isalnum`` / ``str.lower`` (and Final_Sigma) tables (``unicode_tables``), so
  only lines with invalid UTF-8 come back here -- to raise the reference's
  ``UnicodeDecodeError``;
* host (csrc/corpus.cpp, multi-threaded, only when ``backend="host"`` is named --
  the CPU test suite and the bench's comparison leg): pure-ASCII segments natively, segments with
  non-ASCII bytes (whole lines holding U+03A3) tokenized here with the reference's
  rule (``[^\\W_]+`` over ``str.lower()``) and handed back.

Either way the vocabulary order and the documents are exactly the reference's.

``build_corpus_csr`` returns the batch layout the signing path consumes
(int64 indptr + uint32 ids); ``sign_corpus`` is the reference CLI's ``sign``
(cli.py:205-230): ingest, choose the prime, sign every non-empty document on the
GPU and stream the records to the signature file.
"""
from __future__ import annotations

import ctypes as C
import re
import sys
import threading
from fractions import Fraction
from pathlib import Path
from typing import NamedTuple

import numpy as np

from . import _lib
from .minhash import FeatureSet

_TOKEN = re.compile(r"[^\W_]+", re.UNICODE)
_SEGMENT = re.compile(rb"[A-Za-z0-9\x80-\xff]+")  # tokens never cross ASCII separators


def tokenize(text: str) -> tuple[str, ...]:
    """Sorted, deduplicated lowercase terms of one document (reference corpus.py:21-23)."""
    return tuple(sorted(set(_TOKEN.findall(text.lower()))))


class Vocabulary:
    """Bijective term <-> id map; ids run 0..M-1 in first-occurrence order
    (reference corpus.py:26-58)."""

    def __init__(self):
        self._term_to_id: dict[str, int] = {}
        self._id_to_term: list[str] = []

    @classmethod
    def _from_terms(cls, terms: list[str]) -> "Vocabulary":
        v = cls()
        v._id_to_term = terms
        v._term_to_id = None  # built on first lookup
        return v

    def _index(self) -> dict:
        if self._term_to_id is None:
            self._term_to_id = dict(zip(self._id_to_term, range(len(self._id_to_term))))
        return self._term_to_id

    def add(self, term: str) -> int:
        self._index()
        tid = self._term_to_id.get(term)
        if tid is None:
            tid = len(self._id_to_term)
            self._term_to_id[term] = tid
            self._id_to_term.append(term)
        return tid

    def id_of(self, term: str) -> int:
        return self._index()[term]

    def term_of(self, tid: int) -> str:
        return self._id_to_term[tid]

    def __len__(self) -> int:
        return len(self._id_to_term)

    def __contains__(self, term: str) -> bool:
        return term in self._index()

    @property
    def terms(self) -> tuple[str, ...]:
        return tuple(self._id_to_term)


class CorpusData(NamedTuple):
    vocabulary: Vocabulary
    documents: list[FeatureSet]
    empty_documents: int


class CorpusCSR(NamedTuple):
    """The corpus as one CSR batch: document d is ids[indptr[d]:indptr[d+1]] (sorted)."""
    vocabulary: Vocabulary
    indptr: np.ndarray  # int64 [n_docs + 1]
    ids: np.ndarray     # uint32 [nnz]
    empty_documents: int


class _UnicodeTables(C.Structure):  # include/mhb.h mhb_unicode_tables
    _fields_ = [("alnum_bits", C.c_void_p), ("lower_keys", C.c_void_p), ("lower_vals", C.c_void_p),
                ("n_lower", C.c_int32), ("cased_bits", C.c_void_p), ("ignorable_bits", C.c_void_p)]


_UNI: list = []  # (struct, arrays) built once per process


def _bitmap(flags) -> np.ndarray:
    bits = np.fromiter(flags, dtype=bool, count=0x110000)
    return np.ascontiguousarray(np.packbits(bits.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").ravel(),
                                dtype=np.uint32)


def _case_ignorable(c: str, cased: bool) -> bool:
    """Case_Ignorable as THIS Python's str.lower() sees it (its Final_Sigma rule skips such
    code points): probed through the rule itself rather than re-derived."""
    if cased:  # backward scan from a final U+03A3 stops at a cased c unless c is ignorable
        return ("1" + c + "\u03a3").lower()[-1] == "\u03c3"
    return ("A\u03a3" + c + "A").lower()[1] == "\u03c3"


def unicode_tables():
    """str.isalnum / str.lower (and the Cased / Case_Ignorable sets its Final_Sigma rule
    uses) of THIS Python over every code point -- the rules tokenize() applies -- packed
    for mhb_corpus_scan_device (about 1 s, once per process)."""
    if not _UNI:
        chars = [chr(c) for c in range(0x110000)]
        alnum = _bitmap(c.isalnum() for c in chars)
        cased_l = [c.islower() or c.isupper() or c.istitle() for c in chars]
        cased = _bitmap(cased_l)
        ign = _bitmap(_case_ignorable(c, k) for c, k in zip(chars, cased_l))
        keys, vals = [], []
        for c in range(0x80, 0x110000):
            low = chars[c].lower()
            if low != chars[c]:
                if len(low) > 3:
                    raise NotImplementedError(f"lowercase of U+{c:04X} has {len(low)} code points")
                keys.append(c)
                vals.extend([ord(x) for x in low] + [0xFFFFFFFF] * (3 - len(low)))
        k = np.asarray(keys, dtype=np.uint32)
        v = np.asarray(vals, dtype=np.uint32)
        st = _UnicodeTables(alnum.ctypes.data, k.ctypes.data if k.size else None, v.ctypes.data if v.size else None,
                            int(k.size), cased.ctypes.data, ign.ctypes.data)
        _UNI[:] = [st, (alnum, k, v, cased, ign)]
    return _UNI[0]


def _ingest(text, n_bytes: int, threads: int | None, device: int | None, on_device: bool = False) -> CorpusCSR:
    """text: bytes-like host buffer (numpy uint8 / pinned tensor view) of n_bytes."""
    lib = _lib.load()
    buf = text if isinstance(text, np.ndarray) else np.frombuffer(text, dtype=np.uint8)
    if buf.size == 0:
        buf = np.zeros(1, dtype=np.uint8)
    h = C.c_void_p()
    if device is None:
        _lib.check(lib.mhb_corpus_scan(buf.ctypes.data, n_bytes, int(threads or 0), C.byref(h)))
    else:
        _lib.check(lib.mhb_corpus_scan_device(buf.ctypes.data, n_bytes, int(device), C.byref(unicode_tables()),
                                              C.byref(h)))
    try:
        n_docs, n_def = C.c_int64(), C.c_int64()
        _lib.check(lib.mhb_corpus_info(h, C.byref(n_docs), C.byref(n_def)))
        if n_def.value:
            lines = np.empty(n_def.value, dtype=np.int64)
            starts = np.empty_like(lines)
            lens = np.empty_like(lines)
            _lib.check(lib.mhb_corpus_deferred(h, lines.ctypes.data, starts.ctypes.data, lens.ctypes.data))
            line_ptr = np.zeros(n_def.value + 1, dtype=np.int64)
            all_terms = []
            for k in range(n_def.value):
                s = int(starts[k])
                terms = _deferred_terms(buf[s:s + int(lens[k])].tobytes())
                all_terms.extend(terms)
                line_ptr[k + 1] = line_ptr[k] + len(terms)
            # terms never contain "\n": join, encode once, split by the separators in numpy
            joined = np.frombuffer(("\n".join(all_terms) + "\n").encode("utf-8"), dtype=np.uint8)
            nl = np.flatnonzero(joined == 10)
            term_off = np.zeros(nl.size + 1, dtype=np.int64)
            term_off[1:] = nl + 1 - np.arange(1, nl.size + 1)  # starts in the separator-free blob
            blob = joined[joined != 10]
            if not blob.size:
                blob = np.zeros(1, dtype=np.uint8)
            _lib.check(lib.mhb_corpus_set_terms(h, n_def.value, lines.ctypes.data, line_ptr.ctypes.data,
                                                blob.ctypes.data, term_off.ctypes.data))
        nnz, n_terms, tbytes, empty = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(lib.mhb_corpus_intern(h, C.byref(nnz), C.byref(n_terms), C.byref(tbytes), C.byref(empty)))
        tblob = np.empty(max(1, tbytes.value), dtype=np.uint8)
        if on_device:
            import torch

            dev = torch.device("cuda", device)
            indptr = torch.empty(n_docs.value + 1, dtype=torch.int64, device=dev)
            ids = torch.empty(max(1, nnz.value), dtype=torch.uint32, device=dev)[:nnz.value]
            with torch.cuda.device(dev):
                st = torch.cuda.current_stream(dev)
                _lib.check(lib.mhb_corpus_export_device(h, indptr.data_ptr(), ids.data_ptr(), st.cuda_stream))
            _lib.check(lib.mhb_corpus_export(h, None, None, None, tblob.ctypes.data))
        else:
            indptr = np.empty(n_docs.value + 1, dtype=np.int64)
            ids = np.empty(nnz.value, dtype=np.uint32)
            _lib.check(lib.mhb_corpus_export(h, indptr.ctypes.data, ids.ctypes.data, None, tblob.ctypes.data))
    finally:
        lib.mhb_corpus_free(h)
    terms = tblob[:tbytes.value].tobytes().decode("utf-8").split("\n")[:-1] if n_terms.value else []
    return CorpusCSR(Vocabulary._from_terms(terms), indptr, ids, int(empty.value))


def _deferred_terms(line: bytes) -> tuple[str, ...]:
    """The caller's share of a line holding non-ASCII bytes (include/mhb.h): the
    reference's tokenize() over the line's segments that hold non-ASCII bytes (the
    pure-ASCII ones are tokenized natively), or over the whole line when it holds
    U+03A3, whose lowercase (Final_Sigma) depends on context across separators.
    Decoding is strict UTF-8, as open(path, encoding="utf-8") in the reference: every
    byte >= 0x80 sits in a decoded segment."""
    if b"\xce\xa3" in line:
        return tokenize(line.decode("utf-8"))
    return tokenize("\n".join(seg.decode("utf-8") for seg in _SEGMENT.findall(line) if not seg.isascii()))


def _resolve_backend(backend: str, device):
    if backend not in ("gpu", "host"):
        raise ValueError(f"backend must be 'gpu' or 'host', got {backend!r}")
    if backend == "host":
        return None
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("corpus ingest: backend='gpu' needs a visible CUDA device "
                           "(the host ingest is opt-in: backend='host')")
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index or 0


def build_corpus_csr(path_or_bytes, threads: int | None = None, *, backend: str = "gpu", device=None,
                     on_device: bool = False) -> CorpusCSR:
    """Ingest a one-document-per-line UTF-8 file (or its bytes) into a CSR batch.

    Same documents, vocabulary and empty-document tally as ``build_corpus``; the
    rows are the documents' sorted ids, ready for ``signatures_csr``.
    backend: "gpu" (csrc/corpus_gpu.cu, the default) or "host" (csrc/corpus.cpp,
    `threads` workers), named by the caller: nothing is chosen for it.  on_device (GPU backend): indptr / ids
    come back as CUDA tensors instead of numpy arrays."""
    dev = _resolve_backend(backend, device)
    if on_device and dev is None:
        raise ValueError("on_device=True needs the GPU backend")
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        data = np.frombuffer(bytes(path_or_bytes), dtype=np.uint8)
        return _ingest(data, data.size, threads, dev, on_device)
    path = Path(path_or_bytes)
    n = path.stat().st_size
    view = _staging(n) if dev is not None else np.empty(n, dtype=np.uint8)
    _read_parallel(path, view, n)
    return _ingest(view, n, threads, dev, on_device)


def _read_parallel(path, view: np.ndarray, n: int, parts: int = 8, min_part: int = 8 << 20) -> None:
    """Read the file into `view` with concurrent pread calls (the GIL is released
    during each read), so a page-cached file streams at memory-copy speed."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    parts = max(1, min(parts, n // min_part))
    fd = os.open(path, os.O_RDONLY)
    try:
        mv = memoryview(view)

        def read(k):
            lo, hi = n * k // parts, n * (k + 1) // parts
            off = lo
            while off < hi:
                got = os.preadv(fd, [mv[off:hi]], off)
                if got <= 0:
                    raise OSError(f"short read of {path} at byte {off}")
                off += got

        if parts == 1:
            read(0)
        else:
            with ThreadPoolExecutor(parts) as ex:
                list(ex.map(read, range(parts)))
    finally:
        os.close(fd)


_STAGING = threading.local()  # per-thread pinned host buffer, grown on demand (full-speed H2D of the text)


def _staging(n: int) -> np.ndarray:
    import torch

    buf = getattr(_STAGING, "buf", None)
    if buf is None or buf.numel() < n:
        buf = _STAGING.buf = torch.empty(max(n, 1 << 20), dtype=torch.uint8, pin_memory=True)
    return buf.numpy()[:n]


def build_corpus(path, *, backend: str = "gpu") -> CorpusData:
    """Read a one-document-per-line UTF-8 file into id feature sets
    (reference corpus.py:67-80); empty documents are kept and tallied.
    backend: as in build_corpus_csr (the GPU unless "host" is named)."""
    c = build_corpus_csr(path, backend=backend)
    ip, ids = c.indptr, c.ids.astype(np.int64)
    docs = [FeatureSet(ids[ip[d]:ip[d + 1]]) for d in range(ip.size - 1)]
    return CorpusData(c.vocabulary, docs, c.empty_documents)


def synth_pair(j_target: float, size: int, seed: int, id_space: int | None = None):
    """Two random-id sets whose exact Jaccard index is the closest fraction k/u to
    j_target with u <= 2*size (reference corpus.py:83-111)."""
    if not 0.0 < j_target < 1.0:
        raise ValueError(f"target Jaccard must lie in (0, 1), got {j_target}")
    if size < 1:
        raise ValueError(f"size must be positive, got {size}")
    frac = Fraction(j_target).limit_denominator(2 * size)
    k, u = frac.numerator, frac.denominator
    if k == 0:
        raise ValueError(f"target {j_target} is not representable with union size <= {2 * size}")
    if id_space is None:
        id_space = max(64 * size, 1024)
    if id_space < u:
        raise ValueError(f"id space {id_space} too small for union of {u}")
    ids = np.random.default_rng(int(seed)).choice(id_space, size=u, replace=False).astype(np.int64)
    left = (u - k + 1) // 2
    return (FeatureSet(np.concatenate([ids[:k], ids[k:k + left]])),
            FeatureSet(np.concatenate([ids[:k], ids[k + left:]])))


def synth_corpus(n_docs: int, doc_size: int, seed: int, id_space: int | None = None) -> list[FeatureSet]:
    """Random feature sets with sizes jittered +-20% around doc_size
    (reference corpus.py:114-130; CSR form: gen.synth_corpus_numpy)."""
    from .gen import synth_corpus_numpy

    ip, ids = synth_corpus_numpy(n_docs, doc_size, seed, id_space)
    return [FeatureSet(ids[ip[d]:ip[d + 1]]) for d in range(ip.size - 1)]


def sign_corpus(corpus, out, *, family: str, hashes: int = 128, prime: int | None = None, seed: int = 0,
                fmt: str = "text", threads: int | None = None, backend: str = "gpu",
                log=sys.stderr) -> tuple[int, int]:
    """The reference CLI's ``sign`` (cli.py:205-230): ingest `corpus`, build the family,
    sign every non-empty document on the GPU and write (doc_id, signature) records to
    `out` in the reference's text or binary format.  Returns (records, prime)."""
    from .families import make_family
    from .modmath import choose_prime, next_prime
    from .records import write_signatures_csr

    if fmt not in ("text", "binary"):
        raise ValueError(f"fmt must be 'text' or 'binary', got {fmt!r}")
    dev = _resolve_backend(backend, None)
    c = build_corpus_csr(corpus, threads, backend=backend, on_device=dev is not None)
    vocab_size = len(c.vocabulary)
    if vocab_size == 0:
        raise ValueError(f"corpus {corpus} holds no tokens to sign")
    if prime is not None:
        p = next_prime(max(vocab_size, prime, 2))
    else:
        p = choose_prime(vocab_size - 1, hashes)
    fam = make_family(family, seed, hashes, p)
    if dev is not None:  # CSR already resident: drop the empty documents on the device
        import torch

        sizes_t = c.indptr[1:] - c.indptr[:-1]
        keep_t = torch.nonzero(sizes_t > 0).flatten()
        if keep_t.numel() == sizes_t.numel():
            ip, ids, oids = c.indptr, c.ids, None
        else:
            ks = sizes_t[keep_t]
            ip = torch.zeros(keep_t.numel() + 1, dtype=torch.int64, device=sizes_t.device)
            torch.cumsum(ks, 0, out=ip[1:])
            sel = torch.repeat_interleave(keep_t, ks)
            pos = torch.arange(int(ip[-1]), device=ip.device) - torch.repeat_interleave(ip[:-1], ks) + c.indptr[sel]
            ids, oids = c.ids.view(torch.int32)[pos].view(torch.uint32), keep_t.cpu().numpy()
        sizes = sizes_t.cpu().numpy()
        keep = np.flatnonzero(sizes > 0)
    else:
        sizes = np.diff(c.indptr)
        keep = np.flatnonzero(sizes > 0)
        if keep.size == sizes.size:
            ip, ids, oids = c.indptr, c.ids, None
        else:
            ip = np.zeros(keep.size + 1, dtype=np.int64)
            ip[1:] = np.cumsum(sizes[keep])
            sel = np.repeat(keep, sizes[keep])
            pos = np.arange(ip[-1]) - np.repeat(ip[:-1], sizes[keep]) + c.indptr[sel]
            ids, oids = c.ids[pos], keep
    skipped = int(sizes.size - keep.size)
    n = write_signatures_csr(out, ip, ids, fam, fmt=fmt, obj_ids=oids) if keep.size else _touch(out)
    if skipped and log is not None:
        log.write(f"skipped {skipped} empty document(s)\n")
    return n, p


def _touch(path) -> int:
    Path(path).write_bytes(b"")
    return 0


__all__ = ["CorpusCSR", "CorpusData", "Vocabulary", "build_corpus", "build_corpus_csr", "sign_corpus",
           "synth_corpus", "synth_pair", "tokenize"]
