"""Corpus ingest -> CSR, and the reference's ``sign`` command on top of it.

Mirrors ``minhashlab.corpus`` (reference src/corpus.py:18-80): ``tokenize``,
``Vocabulary``, ``CorpusData``, ``build_corpus`` keep their names, arguments and
results.  The work runs in libmhb's native multi-threaded ingest
(csrc/corpus.cpp, ``mhb_corpus_*``): pure-ASCII lines are tokenized and interned
there; lines holding non-ASCII bytes are tokenized here with the reference's Unicode
rule (``[^\\W_]+`` over ``str.lower()``) and handed back, so the vocabulary order and
the documents are exactly the reference's.

``build_corpus_csr`` returns the batch layout the signing path consumes
(int64 indptr + uint32 ids); ``sign_corpus`` is the reference CLI's ``sign``
(cli.py:205-230): ingest, choose the prime, sign every non-empty document on the
GPU and stream the records to the signature file.
"""
from __future__ import annotations

import ctypes as C
import re
import sys
from fractions import Fraction
from pathlib import Path
from typing import NamedTuple

import numpy as np

from . import _lib
from .minhash import FeatureSet

_TOKEN = re.compile(r"[^\W_]+", re.UNICODE)


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
        v._id_to_term = list(terms)
        v._term_to_id = dict(zip(v._id_to_term, range(len(v._id_to_term))))
        return v

    def add(self, term: str) -> int:
        tid = self._term_to_id.get(term)
        if tid is None:
            tid = len(self._id_to_term)
            self._term_to_id[term] = tid
            self._id_to_term.append(term)
        return tid

    def id_of(self, term: str) -> int:
        return self._term_to_id[term]

    def term_of(self, tid: int) -> str:
        return self._id_to_term[tid]

    def __len__(self) -> int:
        return len(self._id_to_term)

    def __contains__(self, term: str) -> bool:
        return term in self._term_to_id

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


def _ingest(text: bytes, threads: int | None) -> CorpusCSR:
    lib = _lib.load()
    buf = np.frombuffer(text, dtype=np.uint8) if len(text) else np.zeros(1, dtype=np.uint8)
    h = C.c_void_p()
    _lib.check(lib.mhb_corpus_scan(buf.ctypes.data, len(text), int(threads or 0), C.byref(h)))
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
                # strict UTF-8, as open(path, encoding="utf-8") in the reference
                terms = tokenize(text[s:s + int(lens[k])].decode("utf-8"))
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
        indptr = np.empty(n_docs.value + 1, dtype=np.int64)
        ids = np.empty(nnz.value, dtype=np.uint32)
        toff = np.empty(n_terms.value + 1, dtype=np.int64)
        tblob = np.empty(max(1, tbytes.value), dtype=np.uint8)
        _lib.check(lib.mhb_corpus_export(h, indptr.ctypes.data, ids.ctypes.data, toff.ctypes.data,
                                         tblob.ctypes.data))
    finally:
        lib.mhb_corpus_free(h)
    terms = tblob[:tbytes.value].tobytes().decode("utf-8").split("\n")[:-1] if n_terms.value else []
    return CorpusCSR(Vocabulary._from_terms(terms), indptr, ids, int(empty.value))


def build_corpus_csr(path_or_bytes, threads: int | None = None) -> CorpusCSR:
    """Ingest a one-document-per-line UTF-8 file (or its bytes) into a CSR batch.

    Same documents, vocabulary and empty-document tally as ``build_corpus``; the
    rows are the documents' sorted ids, ready for ``signatures_csr``."""
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        text = bytes(path_or_bytes)
    else:
        text = Path(path_or_bytes).read_bytes()
    return _ingest(text, threads)


def build_corpus(path) -> CorpusData:
    """Read a one-document-per-line UTF-8 file into id feature sets
    (reference corpus.py:67-80); empty documents are kept and tallied."""
    c = build_corpus_csr(path)
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
                fmt: str = "text", threads: int | None = None, log=sys.stderr) -> tuple[int, int]:
    """The reference CLI's ``sign`` (cli.py:205-230): ingest `corpus`, build the family,
    sign every non-empty document on the GPU and write (doc_id, signature) records to
    `out` in the reference's text or binary format.  Returns (records, prime)."""
    from .families import make_family
    from .modmath import choose_prime, next_prime
    from .records import write_signatures_csr

    if fmt not in ("text", "binary"):
        raise ValueError(f"fmt must be 'text' or 'binary', got {fmt!r}")
    c = build_corpus_csr(corpus, threads)
    vocab_size = len(c.vocabulary)
    if vocab_size == 0:
        raise ValueError(f"corpus {corpus} holds no tokens to sign")
    if prime is not None:
        p = next_prime(max(vocab_size, prime, 2))
    else:
        p = choose_prime(vocab_size - 1, hashes)
    fam = make_family(family, seed, hashes, p)
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
