"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package ``minhashlab`` from /root/reference/pkg/src and
records its outputs -- family parameter draws, signatures (``minhash.signature``),
Jaccard estimates (``estimate_jaccard``) and bucket histograms
(``eval_all(x) % buckets`` + ``bincount``, stats.py:221-224) -- on seeded inputs
as small .npz / .json files next to this script.  The GPU box has no
/root/reference; the committed fixtures travel instead.

Inputs are generated with numpy PCG64 only (``paper_1401_6124_b200.gen.cfg1_numpy``
and local rng calls), so they are reproducible wherever numpy 2.3 runs.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import minhashlab as ref  # noqa: E402  (the reference, read-only)
from minhashlab import corpus as ref_corpus  # noqa: E402

from paper_1401_6124_b200 import gen  # noqa: E402


def ref_sign_csr(indptr, ids, fam):
    out = np.empty((indptr.size - 1, fam.size), dtype=np.int64)
    for s in range(indptr.size - 1):
        fs = ref.FeatureSet(ids[indptr[s]:indptr[s + 1]].astype(np.int64))
        out[s] = ref.signature(fs, fam).mins
    return out


def csr_from_rows(rows):
    sizes = np.array([len(r) for r in rows], dtype=np.int64)
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(sizes, out=indptr[1:])
    ids = np.concatenate([np.asarray(r, dtype=np.int64) for r in rows]) if rows else np.zeros(0, np.int64)
    return indptr, ids.astype(np.uint32)


def families_fixture():
    cases = []
    rng = np.random.default_rng(11)
    for kind in ("random", "iterative"):
        for prime in (7757, 1_048_583, 16_777_259, 4_194_319, 67_108_879, 1_073_741_827):
            for hashes in (1, 128, 2048):
                seed = int(rng.integers(0, 2**63))
                fam = ref.make_family(kind, seed, hashes, prime)
                if kind == "random":
                    a, b = fam.a.copy(), fam.b.copy()
                else:
                    a, b = np.array([fam.base.a]), np.array([fam.base.b])
                cases.append((kind, seed, hashes, prime, a, b))
    # the derived seeds the benchmark configurations use
    derived = {f"cfg{c}_{k}": ref.derive_seed(20260810, c, k) for c in range(1, 6) for k in (0, 1, 100)}
    arrays = {}
    meta = []
    for n, (kind, seed, hashes, prime, a, b) in enumerate(cases):
        arrays[f"a{n}"] = a
        arrays[f"b{n}"] = b
        meta.append({"kind": kind, "seed": seed, "hashes": hashes, "prime": prime})
    np.savez_compressed(HERE / "families.npz", **arrays)
    (HERE / "families.json").write_text(json.dumps({"cases": meta, "derived_seeds": derived}, indent=1))


def fuzz_fixture():
    """Small-prime cases in the style of tests/test_minhash.py:118-129 (own seed)."""
    rng = np.random.default_rng(2026)
    rows, meta, outs = [], [], []
    for case in range(80):
        p = int(rng.choice([11, 31, 101, 7757]))
        size = int(rng.integers(1, min(9, p) if p < 100 else 40))
        ids = rng.choice(p, size=size, replace=False)
        n = int(rng.integers(1, max(2, (p - 3) // 2))) if p < 7757 else int(rng.integers(1, 300))
        kind = ("random", "iterative")[case % 2]
        seed = int(rng.integers(0, 2**62))
        fam = ref.make_family(kind, seed, n, p)
        sig = ref.signature(ref.FeatureSet(ids), fam)
        rows.append(np.sort(ids))
        meta.append({"kind": kind, "seed": seed, "n": n, "p": p})
        outs.append(sig.mins)
    indptr, ids = csr_from_rows(rows)
    out_ptr = np.zeros(len(outs) + 1, dtype=np.int64)
    np.cumsum([o.size for o in outs], out=out_ptr[1:])
    np.savez_compressed(HERE / "fuzz_small.npz", indptr=indptr, ids=ids, out_ptr=out_ptr,
                        out=np.concatenate(outs))
    (HERE / "fuzz_small.json").write_text(json.dumps(meta))


def known_answers():
    ka = {}
    fam = ref.IterativeFamily(3, 5, 7, 1)
    ka["two_element"] = {"a": 3, "b": 5, "p": 7, "n": 1, "ids": [2, 5],
                         "mins": ref.signature(ref.FeatureSet([2, 5]), fam).mins.tolist()}
    ka["iterative_eval_all"] = {"a": 3, "b": 5, "p": 7, "n": 3, "x": 2,
                                "values": ref.IterativeFamily(3, 5, 7, 3).eval_all(2).tolist()}
    sing = {}
    for kind in ("random", "iterative"):
        f = ref.make_family(kind, 3, 16, 7757)
        sing[kind] = ref.signature(ref.FeatureSet([42]), f).mins.tolist()
    ka["singleton_42"] = {"seed": 3, "n": 16, "p": 7757, "mins": sing}
    ka["next_prime_7750"] = ref.next_prime(7750)
    ka["choose_prime"] = {str(v): ref.choose_prime((1 << v) - 1, n) for v, n in
                          ((20, 128), (24, 256), (22, 512), (26, 2048), (30, 256))}
    (HERE / "known_answers.json").write_text(json.dumps(ka, indent=1))


def cfg1_fixture():
    cfg = gen.CONFIGS["cfg1"]
    indptr, ids = gen.cfg1_numpy()
    sub = 400
    arrays = {"indptr_sub": indptr[:sub + 1], "ids_sub": ids[:indptr[sub]]}
    meta = {"n_sets": int(indptr.size - 1), "nnz": int(ids.size),
            "input_sha256": hashlib.sha256(indptr.tobytes() + ids.tobytes()).hexdigest(),
            "prime": cfg.prime, "n_hash": cfg.n_hash}
    for kind in ("random", "iterative"):
        fam = ref.make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
        full = ref_sign_csr(indptr, ids, fam)
        arrays[f"out_sub_{kind}"] = full[:sub]
        meta[f"{kind}_seed"] = cfg.family_seed(kind)
        meta[f"{kind}_sha256"] = hashlib.sha256(np.ascontiguousarray(full, dtype="<i8").tobytes()).hexdigest()
        meta[f"{kind}_sum"] = int(full.sum())
    np.savez_compressed(HERE / "cfg1_sub.npz", **arrays)
    (HERE / "cfg1.json").write_text(json.dumps(meta, indent=1))


def long_sets_fixture():
    """Sets around and far beyond the kernels' 1024-feature chunk, several lane geometries."""
    rng = np.random.default_rng(77)
    sizes = [1, 2, 1023, 1024, 1025, 2047, 2048, 2049, 3000, 5000]
    rows = [np.sort(rng.choice(1 << 20, size=k, replace=False)) for k in sizes]
    indptr, ids = csr_from_rows(rows)
    p = 1_048_583
    arrays = {"indptr": indptr, "ids": ids}
    meta = []
    for n, (kind, hashes) in enumerate((("iterative", 64), ("iterative", 300), ("iterative", 2100),
                                        ("random", 100), ("random", 40), ("iterative", 7))):
        seed = int(rng.integers(0, 2**62))
        fam = ref.make_family(kind, seed, hashes, p)
        arrays[f"out{n}"] = ref_sign_csr(indptr, ids, fam)
        meta.append({"kind": kind, "seed": seed, "n": hashes, "p": p})
    np.savez_compressed(HERE / "long_sets.npz", **arrays)
    (HERE / "long_sets.json").write_text(json.dumps(meta))


def hist_fixture():
    """Reference bucket counts: eval_all(x) % buckets, bincount (stats.py:221-224)."""
    cases = []
    for n, (kind, prime, buckets, hashes) in enumerate((("random", 7757, 100, 1000), ("iterative", 7757, 100, 1000),
                                                          ("iterative", 4_194_319, 4096, 512),
                                                          ("random", 4_194_319, 4096, 512),
                                                          ("iterative", 16_777_259, 64, 256))):
        seed = ref.derive_seed(20260810, 7, n)
        fam = ref.make_family(kind, ref.derive_seed(seed, 0), hashes, prime)
        xrng = np.random.default_rng(ref.derive_seed(seed, 1))
        xs = xrng.integers(0, prime, size=1 if n < 2 else 300)
        counts = np.zeros(buckets, dtype=np.int64)
        for x in xs.tolist():
            counts += np.bincount(fam.eval_all(int(x)) % buckets, minlength=buckets)
        cases.append({"kind": kind, "seed": ref.derive_seed(seed, 0), "hashes": hashes, "prime": prime,
                      "buckets": buckets, "xs": xs.tolist(), "counts": counts.tolist()})
    (HERE / "hist.json").write_text(json.dumps(cases))


def jaccard_fixture():
    """Planted pairs (corpus.synth_pair) -> reference signatures and estimate_jaccard."""
    prime = 4_194_319
    rows, est, exact, meta = [], {}, [], []
    rng = np.random.default_rng(5)
    for k in range(60):
        j = float(rng.uniform(0.1, 0.95))
        s1, s2 = ref_corpus.synth_pair(j, 300, int(rng.integers(0, 2**62)), id_space=1 << 22)
        rows += [s1.ids, s2.ids]
        exact.append(ref.exact_jaccard(s1, s2))
    indptr, ids = csr_from_rows(rows)
    for kind in ("random", "iterative"):
        fam = ref.make_family(kind, 99 if kind == "random" else 100, 512, prime)
        sigs = [ref.signature(ref.FeatureSet(r.astype(np.int64)), fam) for r in rows]
        est[kind] = [ref.estimate_jaccard(sigs[2 * k], sigs[2 * k + 1]) for k in range(len(rows) // 2)]
        meta.append({"kind": kind, "seed": 99 if kind == "random" else 100, "n": 512, "p": prime})
    np.savez_compressed(HERE / "jaccard.npz", indptr=indptr, ids=ids)
    (HERE / "jaccard.json").write_text(json.dumps({"families": meta, "estimates": est, "exact": exact}))


def wide_fixture():
    """Primes >= 2^31: the reference's int64 numba path (p <= MAX_VECTOR_PRIME) and its
    exact `_signature_by_rows` fallback beyond (minhash.py:102-127)."""
    rng = np.random.default_rng(31)
    rows = [np.sort(rng.choice(1 << 31, size=int(k), replace=False)) for k in rng.integers(1, 40, 24)]
    indptr, ids = csr_from_rows(rows)
    arrays = {"indptr": indptr, "ids": ids}
    meta = []
    primes = (ref.next_prime(2**31), ref.next_prime(3_000_000_000), ref.next_prime(3_037_000_500),
              ref.next_prime(2**62))
    n = 0
    for p in primes:
        for kind, hashes in (("iterative", 37), ("random", 19)):
            seed = int(rng.integers(0, 2**62))
            fam = ref.make_family(kind, seed, hashes, p)
            arrays[f"out{n}"] = ref_sign_csr(indptr, ids, fam)
            meta.append({"kind": kind, "seed": seed, "n": hashes, "p": p})
            n += 1
    np.savez_compressed(HERE / "wide.npz", **arrays)
    (HERE / "wide.json").write_text(json.dumps(meta))


def synth_corpus_fixture():
    """The reference's synth_corpus for the C6 timing workload: checksum of its sets."""
    docs = ref_corpus.synth_corpus(500, 100, ref.derive_seed(20260810, 6, 0))
    blob = b"".join(np.asarray(d.ids, dtype=np.int64).tobytes() + b"|" for d in docs)
    meta = {"n_docs": 500, "doc_size": 100, "seed": ref.derive_seed(20260810, 6, 0),
            "sha256": hashlib.sha256(blob).hexdigest(),
            "prime": ref.choose_prime(max(d.max_id for d in docs), 100_000)}
    (HERE / "c6.json").write_text(json.dumps(meta, indent=1))


CORPUS_EDGE_CASES = [
    "",
    "\n",
    "a",
    "a\n",
    "The cat ate the mouse\nThe mouse ate the cheese\n",
    "A-B, a_b; 12ab!\r\nDog dog DOG\rx\r\r\ny\n\n...\nZ",
    "\n\n\n",
    "trailing cr\r",
    "x\ty\x0bz\x0cw\x1cq\u2028r\x00s\n",
    "Stra\u00dfe STRASSE \u0130stanbul \u212a kelvin caf\u00e9 CAF\u00c9 \u00b2 x\u00b2y \u0663\u0664 _a_\n"
    " plain ascii line\n\ufeffbom sep line\n",
    "na\u00efve\nNA\u00cfVE naive\n\u65e5\u672c\u8a9e \u30c6\u30b9\u30c8\n\u0391\u03b2\u03b3 abc\n",
    "\ufb01ne fine FINE\n\u1e9e \u00df ss\nABCDEFGHIJKLMNOPQRSTUVWXYZ abcdefghijklmnopqrstuvwxyz0123456789\n",
    # Final_Sigma looks across ASCII case-ignorables (' and .): whole-line lowercase
    "\u039f\u0394\u039f\u03a3 \u039f\u0394\u039f\u03a3'\u0391 \u0391\u03a3.x \u03a3 x_\u0391\u03a3_y \u03a3\u0391 plain\n",
    "\u201ccurly quotes\u201d don\u2019t \u2014 dashes\u2026 and plain words\n",
    "x\u00a0y abc\u0301def \u212aelvin K k mixed ASCII caf\u00e9 na\u00efve end\n",
]

CORPUS_SYNTH = [  # gen.synth_text_corpus arguments
    {"n_lines": 3000, "seed": 11, "words_per_line": 30.0, "vocab": 5000, "unicode_frac": 0.05},
    {"n_lines": 2000, "seed": 12, "words_per_line": 12.0, "vocab": 800, "unicode_frac": 0.0, "crlf": True},
    {"n_lines": 1500, "seed": 13, "words_per_line": 60.0, "vocab": 20000, "unicode_frac": 0.3,
     "empty_frac": 0.1},
]


def corpus_fixture():
    """Reference build_corpus (corpus.py:67-80) on edge-case texts and seeded synthetic
    corpora, plus the bytes of the reference CLI `sign` output (cli.py:205-230)."""
    import tempfile

    import types

    # the reference CLI imports plots.py -> matplotlib (absent here); `sign` never plots
    if "matplotlib" not in sys.modules:
        mpl = types.ModuleType("matplotlib")
        mpl.use = lambda *a, **k: None
        mpl.pyplot = types.ModuleType("matplotlib.pyplot")
        sys.modules["matplotlib"] = mpl
        sys.modules["matplotlib.pyplot"] = mpl.pyplot
    from minhashlab.cli import main as ref_cli

    cases, arrays = [], {}
    texts = [t.encode("utf-8") for t in CORPUS_EDGE_CASES]
    texts += [gen.synth_text_corpus(**kw) for kw in CORPUS_SYNTH]
    with tempfile.TemporaryDirectory() as tmp:
        for k, data in enumerate(texts):
            path = Path(tmp) / f"c{k}.txt"
            path.write_bytes(data)
            vocab, docs, empty = ref_corpus.build_corpus(path)
            indptr = np.zeros(len(docs) + 1, dtype=np.int64)
            indptr[1:] = np.cumsum([len(d) for d in docs])
            ids = np.concatenate([d.ids for d in docs]) if docs else np.zeros(0, dtype=np.int64)
            arrays[f"indptr{k}"] = indptr
            arrays[f"ids{k}"] = ids.astype(np.int64)
            case = {"sha256": hashlib.sha256(data).hexdigest(), "terms": list(vocab.terms), "empty": empty}
            if k >= len(CORPUS_EDGE_CASES):
                case["synth"] = CORPUS_SYNTH[k - len(CORPUS_EDGE_CASES)]
                sign = {}
                for fam in ("random", "iterative"):
                    for fmt in ("text", "binary"):
                        out = Path(tmp) / f"s{k}_{fam}_{fmt}"
                        rc = ref_cli(["sign", "--corpus", str(path), "--family", fam, "--hashes", "16",
                                      "--seed", "3", "--out", str(out), "--format", fmt])
                        assert rc == 0
                        sign[f"{fam}_{fmt}"] = hashlib.sha256(out.read_bytes()).hexdigest()
                case["sign_hashes16_seed3"] = sign
                case["sign_prime"] = ref.choose_prime(len(vocab) - 1, 16)
            else:
                case["text"] = CORPUS_EDGE_CASES[k]
            cases.append(case)
    np.savez_compressed(HERE / "corpus.npz", **arrays)
    (HERE / "corpus.json").write_text(json.dumps(cases, indent=1, ensure_ascii=True))

def wide_ids_fixture():
    """int64 feature ids beyond 2^32 under primes >= 2^32 (the reference's FeatureSet
    is int64; signature() takes _signature_by_rows there, minhash.py:102-127)."""
    rng = np.random.default_rng(2026)
    cases, arrays = [], {}
    for k, (kind, p, n) in enumerate([("iterative", 4_294_967_311, 16), ("random", 4_294_967_311, 12),
                                       ("iterative", 2**62 + 135, 16), ("random", 2**62 + 135, 9)]):
        seed = int(rng.integers(1 << 30))
        fam = ref.make_family(kind, seed, n, p)
        sizes = [1, 2, 7, 40, 13]
        rows = [np.unique(rng.integers(0, p, size=m, dtype=np.int64)) for m in sizes]
        # every case reaches past 2^32: 2^32 itself and the largest ids below p
        rows[1] = np.unique(np.concatenate([rows[1], [2**32, p - 1]]))
        rows[3] = np.unique(np.concatenate([rows[3], [2**32 + 1, p - 2, 7]]))
        indptr = np.zeros(len(rows) + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([r.size for r in rows])
        out = np.stack([ref.signature(ref.FeatureSet(r), fam).mins for r in rows])
        arrays[f"indptr{k}"] = indptr
        arrays[f"ids{k}"] = np.concatenate(rows)
        arrays[f"out{k}"] = out
        cases.append({"kind": kind, "p": p, "n": n, "seed": seed})
    np.savez_compressed(HERE / "wide_ids.npz", **arrays)
    (HERE / "wide_ids.json").write_text(json.dumps(cases, indent=1))


if __name__ == "__main__":
    wide_ids_fixture()
    corpus_fixture()
    synth_corpus_fixture()
    wide_fixture()
    families_fixture()
    known_answers()
    fuzz_fixture()
    long_sets_fixture()
    hist_fixture()
    jaccard_fixture()
    cfg1_fixture()
    print("golden fixtures written to", HERE)
