"""Synthetic workload generators: shapes, canonical sets, determinism (CPU only)."""
import hashlib
import json

import numpy as np
import torch

from paper_1401_6124_b200 import gen


def _check_csr(indptr, ids, vocab):
    ip = indptr.cpu().numpy() if torch.is_tensor(indptr) else indptr
    x = ids.cpu().numpy().astype(np.int64) if torch.is_tensor(ids) else ids.astype(np.int64)
    assert ip[0] == 0 and np.all(np.diff(ip) >= 1) and ip[-1] == x.size
    assert x.min() >= 0 and x.max() < vocab
    for s in range(0, ip.size - 1, max(1, (ip.size - 1) // 200)):
        row = x[ip[s]:ip[s + 1]]
        assert np.all(np.diff(row) > 0), "sets are sorted and duplicate-free"
    return ip, x


def test_cfg1_numpy_matches_golden_input(golden):
    meta = json.loads((golden / "cfg1.json").read_text())
    indptr, ids = gen.cfg1_numpy()
    assert hashlib.sha256(indptr.tobytes() + ids.tobytes()).hexdigest() == meta["input_sha256"]
    ip, _ = _check_csr(indptr, ids, 1 << 20)
    sizes = np.diff(ip)
    assert abs(sizes.mean() - 50) < 1.0


def test_cfg2_shape_small():
    ip, ids = gen.make_csr("cfg2", device="cpu", n_sets=4000)
    ip, x = _check_csr(ip, ids, 1 << 24)
    sizes = np.diff(ip)
    assert 100 < np.median(sizes) < 140  # lognormal median 120
    assert sizes.max() <= 20_000
    # Zipf: the scrambled rank-1 id (0) is the most frequent feature
    assert np.bincount(x).argmax() == 0


def test_make_csr_deterministic():
    a = gen.make_csr("cfg1", device="cpu", n_sets=300, seed=5)
    b = gen.make_csr("cfg1", device="cpu", n_sets=300, seed=5)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1].to(torch.int64), b[1].to(torch.int64))


def test_poisson_configs():
    for name in ("cfg3", "cfg4"):
        cfg = gen.CONFIGS[name]
        ip, ids = gen.make_csr(cfg, device="cpu", n_sets=500)
        ip, _ = _check_csr(ip, ids, cfg.vocab)
        assert abs(np.diff(ip).mean() - cfg.size_a) < 0.1 * cfg.size_a


def test_synth_corpus_matches_reference(golden):
    """gen.synth_corpus_numpy reproduces the reference's synth_corpus sets exactly."""
    meta = json.loads((golden / "c6.json").read_text())
    indptr, ids = gen.synth_corpus_numpy(meta["n_docs"], meta["doc_size"], meta["seed"])
    blob = b"".join(ids[indptr[s]:indptr[s + 1]].astype(np.int64).tobytes() + b"|" for s in range(indptr.size - 1))
    assert hashlib.sha256(blob).hexdigest() == meta["sha256"]
    _, _, prime, _ = gen.c6_workload()
    assert prime == meta["prime"]
