"""Randomized differential stress of the corpus ingest (both backends) against the
pure-Python oracle (oracle/corpus_oracle.py, itself pinned to the reference's output).

usage: python tools/stress_corpus.py [seconds] [seed]

Each case draws a text mix: ASCII words, separators and every line-break kind; the
fuzz alphabet (Final_Sigma contexts, case-expanding and non-alphanumeric code points);
runs of code points from one random Unicode block (scripts stay together, as in real
text); sometimes a few random code points from any plane; and, in some cases, an
invalid UTF-8 sequence (both sides must raise UnicodeDecodeError).  The device backend
(when a GPU is visible) and the host backend (1 or 3 threads) must equal the oracle
exactly: vocabulary order, documents, empty-line tally.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import corpus_oracle  # noqa: E402
from paper_1401_6124_b200.corpus import build_corpus_csr  # noqa: E402

BAD = [b"\xff", b"\xc3\x28", b"\xed\xa0\x80", b"\xf4\x90\x80\x80", b"\xe2\x82", b"\xc0\xaf", b"\x80"]


def _cp(rng, lo, hi):
    while True:
        c = int(rng.integers(lo, hi))
        if not 0xD800 <= c <= 0xDFFF:
            return chr(c)


def make_text(rng):
    n = int(rng.choice([1, 10, 200, 3000, 20000]))
    block = int(rng.integers(0x80, 0x30000)) & ~0xFF
    if 0xD800 <= block <= 0xDFFF:  # no scalar values in the surrogate blocks
        block = 0x80
    out = []
    while len(out) < n:
        r = rng.random()
        if r < 0.35:
            w = int(rng.integers(1, 9))
            out.append("".join(chr(int(c)) for c in rng.integers(0x61, 0x7B, size=w)))
            if rng.random() < 0.2:
                out[-1] = out[-1].upper()
        elif r < 0.5:
            out.append(" \t.,'-_:;"[int(rng.integers(0, 9))])
        elif r < 0.55:
            out.append(["\n", "\r\n", "\r", "\x0b", "\x0c", " ", "\x85"][int(rng.integers(0, 7))])
        elif r < 0.7:
            out.append(corpus_oracle.FUZZ_ALPHABET[int(rng.integers(0, len(corpus_oracle.FUZZ_ALPHABET)))])
        elif r < 0.95:
            out.append("".join(_cp(rng, block, block + 0x100) for _ in range(int(rng.integers(1, 6)))))
        else:
            out.append(_cp(rng, 0x80, 0x110000))
    data = "".join(out).encode("utf-8")
    if rng.random() < 0.05:
        k = int(rng.integers(0, len(data) + 1))
        data = data[:k] + BAD[int(rng.integers(0, len(BAD)))] + data[k:]
    return data


def _run(fn):
    try:
        return fn()
    except UnicodeDecodeError:
        return "UnicodeDecodeError"


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    import torch

    backends = (["gpu"] if torch.cuda.is_available() else []) + ["host"]
    rng = np.random.default_rng(seed)
    t0, n, bad, n_bytes, n_invalid = time.time(), 0, 0, 0, 0
    while time.time() - t0 < seconds:
        data = make_text(rng)
        want = _run(lambda: corpus_oracle.build_corpus_bytes(data))
        n_invalid += want == "UnicodeDecodeError"
        for be in backends:
            threads = 1 if be == "gpu" else int(rng.choice([1, 3]))
            got = _run(lambda: build_corpus_csr(data, threads=threads, backend=be))
            if isinstance(want, str) or isinstance(got, str):
                ok = isinstance(want, str) and isinstance(got, str)
            else:
                terms, ip, x, empty = want
                ok = (list(got.vocabulary.terms) == terms and got.empty_documents == empty
                      and np.array_equal(got.indptr, ip) and np.array_equal(got.ids.astype(np.int64), x))
            if not ok:
                bad += 1
                print("MISMATCH", be, n, len(data), data[:200], flush=True)
        n += 1
        n_bytes += len(data)
    print(f"stress_corpus: {n} texts ({n_bytes / 1e6:.1f} MB, {n_invalid} invalid UTF-8), backends {backends}, "
          f"{bad} mismatches in {time.time() - t0:.0f} s (seed {seed})")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
