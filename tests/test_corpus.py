"""Corpus ingest (reference corpus.py:18-80) through libmhb's native host ingest (CPU only;
named explicitly: backend="host" -- the default is the GPU, tests/test_gpu_parity.py).

The golden fixture (tests/golden/corpus.{json,npz}, made by make_golden.py) holds the
reference's own build_corpus output -- vocabulary order, documents, empty tally --
for edge-case texts (universal newlines, Unicode case folding and alphanumerics,
BOM, NUL, vertical tab / form feed / U+2028 inside lines) and seeded synthetic
corpora.  The unit cases restate the reference's tests/test_corpus.py.
"""
import ctypes as C
import hashlib
import json

import numpy as np
import pytest

from paper_1401_6124_b200 import _lib, gen
from paper_1401_6124_b200.corpus import (Vocabulary, build_corpus, build_corpus_csr, synth_corpus, synth_pair,
                                         tokenize)
from paper_1401_6124_b200.minhash import exact_jaccard

D1 = "The cat ate the mouse"
D2 = "The mouse ate the cheese"


def _cases(golden):
    cases = json.loads((golden / "corpus.json").read_text())
    z = np.load(golden / "corpus.npz")
    for k, case in enumerate(cases):
        data = case["text"].encode("utf-8") if "text" in case else gen.synth_text_corpus(**case["synth"])
        assert hashlib.sha256(data).hexdigest() == case["sha256"]
        yield k, data, case, z[f"indptr{k}"], z[f"ids{k}"]


# --- reference tests/test_corpus.py, restated -----------------------------------------

def test_tokenize_examples():
    assert tokenize(D1) == ("ate", "cat", "mouse", "the")
    assert tokenize(D2) == ("ate", "cheese", "mouse", "the")
    assert tokenize("") == ()
    assert tokenize("  \t .,;!  ") == ()
    assert tokenize("A-B, a_b; 12ab!") == ("12ab", "a", "b")
    assert tokenize("Dog dog DOG") == ("dog",)


def test_vocabulary():
    v = Vocabulary()
    assert [v.add(t) for t in ("b", "a", "b", "c")] == [0, 1, 0, 2]
    assert v.terms == ("b", "a", "c")
    assert v.id_of(v.term_of(1)) == 1
    with pytest.raises(KeyError):
        v.id_of("missing")
    with pytest.raises(IndexError):
        v.term_of(5)
    assert "a" in v and "missing" not in v


def test_build_corpus_worked_pair(tmp_path):
    path = tmp_path / "docs.txt"
    path.write_text(f"{D1}\n{D2}\n", encoding="utf-8")
    vocab, docs, empty = build_corpus(path, backend="host")
    assert len(vocab) == 5 and len(docs) == 2 and empty == 0
    assert exact_jaccard(docs[0], docs[1]) == pytest.approx(3 / 5)


def test_build_corpus_empty_duplicates_blank(tmp_path):
    path = tmp_path / "empty.txt"
    path.write_text("", encoding="utf-8")
    vocab, docs, empty = build_corpus(path, backend="host")
    assert len(vocab) == 0 and docs == [] and empty == 0
    path.write_text(f"{D1}\n{D1}\n", encoding="utf-8")
    _, docs, _ = build_corpus(path, backend="host")
    assert docs[0] == docs[1]
    path.write_text(f"{D1}\n\n...\n{D2}\n", encoding="utf-8")
    _, docs, empty = build_corpus(path, backend="host")
    assert len(docs) == 4 and empty == 2 and len(docs[1]) == 0 and len(docs[2]) == 0


def test_synth_pair_and_corpus():
    a, b = synth_pair(0.5, 40, seed=3)
    assert exact_jaccard(a, b) == pytest.approx(0.5)
    docs = synth_corpus(5, 12, seed=0, id_space=256)
    assert len(docs) == 5 and all(9 <= len(d) <= 15 for d in docs)
    with pytest.raises(ValueError):
        synth_pair(0.0, 10, seed=0)


# --- golden: the reference's own build_corpus output ----------------------------------

@pytest.mark.parametrize("threads", [1, 3, 8])
def test_golden_corpora(golden, threads):
    for k, data, case, indptr, ids in _cases(golden):
        c = build_corpus_csr(data, threads=threads, backend="host")
        assert list(c.vocabulary.terms) == case["terms"], k
        assert c.empty_documents == case["empty"], k
        assert np.array_equal(c.indptr, indptr), k
        assert np.array_equal(c.ids.astype(np.int64), ids), k


def test_golden_build_corpus_feature_sets(golden, tmp_path):
    for k, data, case, indptr, ids in _cases(golden):
        path = tmp_path / f"c{k}.txt"
        path.write_bytes(data)
        vocab, docs, empty = build_corpus(path, backend="host")
        assert list(vocab.terms) == case["terms"] and empty == case["empty"]
        assert len(docs) == indptr.size - 1
        for d in range(0, len(docs), max(1, len(docs) // 50)):
            assert np.array_equal(docs[d].ids, ids[indptr[d]:indptr[d + 1]])


def test_threads_invariant_large():
    text = gen.synth_text_corpus(30000, 5, vocab=50000, unicode_frac=0.02)
    a = build_corpus_csr(text, threads=1, backend="host")
    for t in (2, 7, 16):
        b = build_corpus_csr(text, threads=t, backend="host")
        assert a.vocabulary.terms == b.vocabulary.terms
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.ids, b.ids)


def test_invalid_utf8_raises_like_the_reference():
    with pytest.raises(UnicodeDecodeError):
        build_corpus_csr(b"fine line\nbad \xff\xfe bytes\n", backend="host")


def test_abi_deferred_protocol_errors():
    lib = _lib.load()
    text = np.frombuffer(b"ascii only\ncaf\xc3\xa9 line\n", dtype=np.uint8)
    h = C.c_void_p()
    assert lib.mhb_corpus_scan(text.ctypes.data, text.size, 1, C.byref(h)) == 0
    try:
        nd, nf = C.c_int64(), C.c_int64()
        assert lib.mhb_corpus_info(h, C.byref(nd), C.byref(nf)) == 0
        assert (nd.value, nf.value) == (2, 1)
        # interning before the deferred line's terms arrive is an error
        assert lib.mhb_corpus_intern(h, None, None, None, None) == _lib.MHB_ERR_INVALID
        assert b"deferred" in lib.mhb_last_error()
        # line 0 is native, not deferred
        lines = np.array([0], dtype=np.int64)
        ptr = np.array([0, 0], dtype=np.int64)
        assert lib.mhb_corpus_set_terms(h, 1, lines.ctypes.data, ptr.ctypes.data, None,
                                        ptr.ctypes.data) == _lib.MHB_ERR_INVALID
        assert lib.mhb_corpus_export(h, None, None, None, None) == _lib.MHB_ERR_INVALID
    finally:
        lib.mhb_corpus_free(h)


def test_corpus_oracle_pinned_to_reference(golden):
    """The pure-Python restatement (oracle/corpus_oracle.py) reproduces the reference's
    golden output before it is used as the fuzz checker."""
    from oracle import corpus_oracle

    for k, data, case, indptr, ids in _cases(golden):
        terms, ip, x, empty = corpus_oracle.build_corpus_bytes(data)
        assert terms == case["terms"] and empty == case["empty"], k
        assert np.array_equal(ip, indptr) and np.array_equal(x, ids), k


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_host_backend_against_oracle(seed):
    """Random text over separators, every line-break kind, Final_Sigma contexts and
    case-expanding / non-alphanumeric code points: native ingest == the oracle."""
    from oracle import corpus_oracle

    data = corpus_oracle.fuzz_text(seed, 4000 + 500 * seed)
    terms, ip, x, empty = corpus_oracle.build_corpus_bytes(data)
    for threads in (1, 3):
        c = build_corpus_csr(data, threads=threads, backend="host")
        assert list(c.vocabulary.terms) == terms and c.empty_documents == empty
        assert np.array_equal(c.indptr, ip) and np.array_equal(c.ids.astype(np.int64), x)


def test_gpu_backend_is_the_default_and_never_falls_back(monkeypatch):
    """No dispatch: the default ingest is the GPU's, and without a visible device it
    raises instead of quietly running the host code."""
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="backend='gpu'"):
        build_corpus_csr(b"a b c\n")
    with pytest.raises(ValueError):
        build_corpus_csr(b"a b c\n", backend="auto")
