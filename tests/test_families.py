"""Host-side family construction mirrors the reference exactly (CPU only).

tests/golden/families.npz holds (a, b) drawn by the reference's own
make_family for 36 (kind, seed, hashes, prime) cases; derived seeds come from
the reference's derive_seed.  The remaining checks restate the reference's
family tests (test_families.py:55-225) against this package.
"""
import json

import numpy as np
import pytest

from paper_1401_6124_b200 import (
    IterativeFamily,
    RandomFamily,
    choose_prime,
    derive_seed,
    family_from_json,
    family_to_json,
    is_prime,
    make_family,
    make_iterative_family,
    next_prime,
    sample_random_family,
)
from paper_1401_6124_b200.gen import CONFIGS


def test_parameter_draws_match_reference(golden):
    meta = json.loads((golden / "families.json").read_text())
    z = np.load(golden / "families.npz")
    for n, case in enumerate(meta["cases"]):
        fam = make_family(case["kind"], case["seed"], case["hashes"], case["prime"])
        if case["kind"] == "random":
            assert np.array_equal(fam.a, z[f"a{n}"]) and np.array_equal(fam.b, z[f"b{n}"]), case
        else:
            assert (fam.base.a, fam.base.b) == (int(z[f"a{n}"][0]), int(z[f"b{n}"][0])), case


def test_derived_seeds_match_reference(golden):
    derived = json.loads((golden / "families.json").read_text())["derived_seeds"]
    for key, val in derived.items():
        cfg, k = key.split("_")
        assert derive_seed(20260810, int(cfg[3:]), int(k)) == val


def test_config_primes_match_reference_choose_prime(golden):
    ka = json.loads((golden / "known_answers.json").read_text())
    assert next_prime(7750) == ka["next_prime_7750"] == 7753
    for v, n in ((20, 128), (24, 256), (22, 512), (26, 2048), (30, 256)):
        assert choose_prime((1 << v) - 1, n) == ka["choose_prime"][str(v)]
    assert CONFIGS["cfg2"].prime == 16_777_259 and CONFIGS["cfg5"].prime == 1_073_741_827


def test_validation_errors():
    with pytest.raises(ValueError):
        make_family("tabulation", 0, 2, 7757)
    with pytest.raises(ValueError):
        make_iterative_family(5, 5, 11)  # prime <= 2*hashes + 2
    assert make_iterative_family(5, 5, 13).size == 5
    with pytest.raises(ValueError):
        IterativeFamily(7918, 7918, 7919, 4000)
    with pytest.raises(ValueError):
        sample_random_family(0, 0, 7757)
    with pytest.raises(ValueError):
        sample_random_family(0, 4, 7758)  # not prime
    with pytest.raises(ValueError):
        RandomFamily([0], [0], 7757)
    fam = make_iterative_family(3, 10, 7757)
    with pytest.raises(IndexError):
        fam.eval_at(5, 10)
    with pytest.raises(ValueError):
        fam.eval_all(7757)


def test_closed_form_equals_recurrence():
    rng = np.random.default_rng(99)
    for _ in range(200):
        p = int(rng.choice([31, 7757, 1000003]))
        n = int(rng.integers(1, 60))
        if p <= 2 * n + 2:
            continue
        fam = make_iterative_family(int(rng.integers(0, 2**63)), n, p)
        x = int(rng.integers(0, p))
        a, b = fam.base.a, fam.base.b
        h, walk = (a * x) % p, []
        for _i in range(n):
            walk.append(h)
            h = (h + (x + b) % p) % p
        assert fam.eval_all(x).tolist() == walk == [fam.eval_at(x, i) for i in range(n)]


def test_known_eval_all(golden):
    ka = json.loads((golden / "known_answers.json").read_text())["iterative_eval_all"]
    assert IterativeFamily(ka["a"], ka["b"], ka["p"], ka["n"]).eval_all(ka["x"]).tolist() == ka["values"]


def test_members_are_bijections():
    p = 101
    for fam in (make_iterative_family(4, 20, p), sample_random_family(4, 20, p)):
        table = np.stack([fam.eval_all(x) for x in range(p)])
        for i in range(fam.size):
            assert len(set(table[:, i].tolist())) == p


def test_json_round_trip():
    for kind in ("random", "iterative"):
        fam = make_family(kind, 123, 64, 7757)
        back = family_from_json(family_to_json(fam))
        assert back.key == fam.key
    with pytest.raises(ValueError):
        family_to_json(IterativeFamily(3, 5, 7, 1))
    with pytest.raises(ValueError):
        family_from_json('{"kind": "random"}')


def test_primality():
    assert [n for n in range(50) if is_prime(n)] == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47]
    assert is_prime(2**61 - 1) and not is_prime(3215031751)  # strong pseudoprime to bases 2,3,5,7
    with pytest.raises(ValueError):
        next_prime(1)
