"""CPU oracle for the corpus ingest: a pure-Python restatement of the reference's
``build_corpus`` / ``tokenize`` / ``Vocabulary`` (src/corpus.py:18-80).

TEST INFRASTRUCTURE ONLY -- like oracle.py, it may be imported by tests/ (and
bench.py's CPU arm), never by the product path.

  * lines: text-mode iteration of the UTF-8 file (universal newlines: "\\n",
    "\\r\\n", "\\r"), corpus.py:74-75;
  * terms: sorted(set(re.findall(r"[^\\W_]+", line.lower()))), corpus.py:21-23;
  * ids: Vocabulary.add in (line, sorted term) order, first occurrence wins,
    corpus.py:29-37;
  * documents: FeatureSet(ids) -> sorted unique ids, minhash.py:30-39.
Pinned against the reference itself by tests/golden/corpus.* (test_corpus.py).
"""
from __future__ import annotations

import io
import re

import numpy as np

_TOKEN = re.compile(r"[^\W_]+", re.UNICODE)


def build_corpus_bytes(data: bytes):
    """(terms list in id order, indptr int64, ids int64, empty document count)."""
    vocab: dict[str, int] = {}
    rows, empty = [], 0
    for line in io.TextIOWrapper(io.BytesIO(data), encoding="utf-8"):
        terms = sorted(set(_TOKEN.findall(line.lower())))
        if not terms:
            empty += 1
        ids = []
        for t in terms:
            if t not in vocab:
                vocab[t] = len(vocab)
            ids.append(vocab[t])
        rows.append(sorted(ids))
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    ids = np.fromiter((x for r in rows for x in r), dtype=np.int64, count=int(indptr[-1]))
    return list(vocab), indptr, ids, empty


FUZZ_ALPHABET = (list("abcXYZ019") + [" ", "  ", "'", ".", "_", "-", "\t", "\r", "\n", "\r\n", "\x0b", "\x0c"]
                 + ["Σ", "σ", "ς", "Α", "İ", "K", "é", "É", "́",
                    " ", "“", "’", "ß", "ﬁ", "日", "٣", "²", " ",
                    "﻿", "ẞ"])


def fuzz_text(seed: int, n_chars: int) -> bytes:
    """Seeded random text over FUZZ_ALPHABET (ASCII separators, line breaks of every
    kind, Final_Sigma contexts, case-expanding and non-alphanumeric code points)."""
    rng = np.random.default_rng(seed)
    w = np.array([6.0] * 9 + [3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0.3, 0.3] + [0.6] * 20)
    w /= w.sum()
    picks = rng.choice(len(FUZZ_ALPHABET), size=n_chars, p=w)
    return "".join(FUZZ_ALPHABET[i] for i in picks).encode("utf-8")
