"""Pin the CPU oracle against the reference's own outputs and known answers (CPU only).

The fixtures under tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py); the known-answer vectors come from the
reference's tests (test_minhash.py:83-94, test_families.py:116-120).
"""
import hashlib
import json

import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import IterativeFamily, gen, make_family


def test_known_answer_two_element(golden):
    ka = json.loads((golden / "known_answers.json").read_text())["two_element"]
    out = oracle.sign_iterative_csr([0, 2], [2, 5], ka["a"], ka["b"], ka["p"], ka["n"])
    assert out[0].tolist() == ka["mins"] == [5]


def test_known_answer_eval_all(golden):
    ka = json.loads((golden / "known_answers.json").read_text())["iterative_eval_all"]
    fam = IterativeFamily(ka["a"], ka["b"], ka["p"], ka["n"])
    assert oracle.member_values(fam, ka["x"]).tolist() == ka["values"] == [6, 6, 6]


def test_known_answer_singleton(golden):
    ka = json.loads((golden / "known_answers.json").read_text())["singleton_42"]
    for kind in ("random", "iterative"):
        fam = make_family(kind, ka["seed"], ka["n"], ka["p"])
        out = oracle.sign_family_csr([0, 1], [42], fam)
        assert out[0].tolist() == ka["mins"][kind] == [42] * ka["n"]


def test_fuzz_small_primes(golden):
    z = np.load(golden / "fuzz_small.npz")
    meta = json.loads((golden / "fuzz_small.json").read_text())
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        ip = z["indptr"][k:k + 2]
        got = oracle.sign_family_csr(ip, z["ids"], fam)[0]
        want = z["out"][z["out_ptr"][k]:z["out_ptr"][k + 1]]
        assert np.array_equal(got, want), m
        # and the brute-force restatement of tests/test_minhash.py:27-39
        assert np.array_equal(oracle.brute_force_row(z["ids"][ip[0]:ip[1]], fam), want), m


def test_long_sets(golden):
    z = np.load(golden / "long_sets.npz")
    meta = json.loads((golden / "long_sets.json").read_text())
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        assert np.array_equal(oracle.sign_family_csr(z["indptr"], z["ids"], fam), z[f"out{k}"]), m


def test_cfg1_subsample(golden):
    z = np.load(golden / "cfg1_sub.npz")
    meta = json.loads((golden / "cfg1.json").read_text())
    for kind in ("random", "iterative"):
        fam = make_family(kind, meta[f"{kind}_seed"], meta["n_hash"], meta["prime"])
        got = oracle.sign_family_csr(z["indptr_sub"], z["ids_sub"], fam)
        assert np.array_equal(got, z[f"out_sub_{kind}"])


def test_cfg1_full_checksum(golden):
    """Full cfg1 (10k sets, N=128): the oracle's output hashes to the reference's."""
    meta = json.loads((golden / "cfg1.json").read_text())
    indptr, ids = gen.cfg1_numpy()
    assert hashlib.sha256(indptr.tobytes() + ids.tobytes()).hexdigest() == meta["input_sha256"]
    for kind in ("random", "iterative"):
        fam = make_family(kind, meta[f"{kind}_seed"], meta["n_hash"], meta["prime"])
        out = oracle.sign_family_csr(indptr, ids, fam)
        assert hashlib.sha256(out.astype("<i8").tobytes()).hexdigest() == meta[f"{kind}_sha256"]


def test_histogram_restatement(golden):
    for case in json.loads((golden / "hist.json").read_text()):
        fam = make_family(case["kind"], case["seed"], case["hashes"], case["prime"])
        got = oracle.bucket_histogram(fam, case["xs"], case["buckets"])
        assert got.tolist() == case["counts"]


def test_jaccard_restatement(golden):
    z = np.load(golden / "jaccard.npz")
    meta = json.loads((golden / "jaccard.json").read_text())
    for fm in meta["families"]:
        fam = make_family(fm["kind"], fm["seed"], fm["n"], fm["p"])
        sig = oracle.sign_family_csr(z["indptr"], z["ids"], fam)
        est = [oracle.jaccard_estimate(sig[2 * k], sig[2 * k + 1]) for k in range(sig.shape[0] // 2)]
        assert est == meta["estimates"][fm["kind"]]


@pytest.mark.parametrize("threads", [1, 4])
def test_oracle_thread_count_invariant(threads):
    indptr, ids = gen.cfg1_numpy(n_sets=300, seed=5)
    fam = make_family("iterative", 1, 64, 1_048_583)
    a = oracle.sign_family_csr(indptr, ids, fam, threads=threads)
    b = oracle.sign_family_csr(indptr, ids, fam, threads=1)
    assert np.array_equal(a, b)


def test_wide_primes_restatement(golden):
    """Reference outputs for primes >= 2^31 (incl. its exact fallback beyond 3.04e9)
    equal the Python-int brute force (test_minhash.py:27-39)."""
    z = np.load(golden / "wide.npz")
    meta = json.loads((golden / "wide.json").read_text())
    ip, ids = z["indptr"], z["ids"]
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        for s in range(ip.size - 1):
            assert np.array_equal(oracle.brute_force_row(ids[ip[s]:ip[s + 1]], fam), z[f"out{k}"][s]), m


def test_c_oracle_wide_primes_against_reference(golden):
    """The C oracle itself on the reference's wide-prime outputs: int64 loops up to
    MAX_VECTOR_PRIME, the exact (_signature_by_rows) arithmetic beyond it."""
    z = np.load(golden / "wide.npz")
    meta = json.loads((golden / "wide.json").read_text())
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        if fam.prime >= 1 << 63:
            continue
        assert np.array_equal(oracle.sign_family_csr(z["indptr"], z["ids"], fam), z[f"out{k}"]), m


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_c_oracle_exact_beyond_max_vector_prime(kind):
    """p just below 2^32 (a*x overflows int64): the C oracle == Python-int brute force."""
    rng = np.random.default_rng(5)
    p = 4_294_967_291
    fam = make_family(kind, 11, 9, p)
    ids = np.unique(rng.integers(0, p, size=300)).astype(np.uint32)
    got = oracle.sign_family_csr(np.array([0, ids.size]), ids, fam)[0]
    assert np.array_equal(got, oracle.brute_force_row(ids, fam))


def test_wide_ids_restatement(golden):
    """int64 ids beyond 2^32 (primes >= 2^32): the reference's outputs == brute force."""
    z = np.load(golden / "wide_ids.npz")
    for k, m in enumerate(json.loads((golden / "wide_ids.json").read_text())):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        ip, ids = z[f"indptr{k}"], z[f"ids{k}"]
        assert ids.max() > 2**32
        for s in range(ip.size - 1):
            assert np.array_equal(oracle.brute_force_row(ids[ip[s]:ip[s + 1]], fam), z[f"out{k}"][s]), m


def test_band_key_definition_scalar():
    """oracle.band_keys (vectorised) against a scalar restatement of the band-key
    definition in include/mhb.h / csrc/bandhash.cuh (the reference defines no banding)."""
    M, M64 = 2**32, 2**64

    def key(row, band):
        h1, h2 = 0x811C9DC5 ^ band, 0xC2B2AE35 ^ ((band * 0x27D4EB2F) % M)
        for x in row:
            h1, h2 = (h1 * 0x9E3779B1 + int(x)) % M, (h2 * 0x85EBCA6B + int(x)) % M
        z = ((h1 << 32) | h2) + 0x9E3779B97F4A7C15
        z %= M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % M64
        return z ^ (z >> 31)

    rng = np.random.default_rng(3)
    for rows in (4, 16):
        sig = rng.integers(0, 2**32, size=(7, 4 * rows), dtype=np.uint64)
        got = oracle.band_keys(sig, rows)
        want = [[key(sig[s, b * rows:(b + 1) * rows], b) for b in range(4)] for s in range(7)]
        assert [[int(v) for v in r] for r in got] == want
