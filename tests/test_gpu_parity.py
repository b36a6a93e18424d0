"""GPU parity: libmhb kernels (through the C ABI) against the reference's outputs.

Small cases compare with golden fixtures produced by the reference itself and with
the CPU oracle (pinned in test_oracle.py).  Full-size cases use size-independent
properties: checksums against the reference's full cfg1 output, oracle agreement on
seeded subsamples, argmins drawn from their own sets, and order invariance.
Bar: bit-exact (integer path).
"""
import hashlib
import json

import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import (
    FeatureSet,
    band_keys,
    IterativeFamily,
    RandomFamily,
    bucket_histogram,
    estimate_jaccard,
    estimate_pairs,
    gen,
    jaccard_block,
    make_family,
    signature,
    signatures,
    signatures_band_keys,
    signatures_csr,
)

pytestmark = pytest.mark.gpu


def _dev(indptr, ids, device):
    import torch

    return (torch.as_tensor(np.asarray(indptr, dtype=np.int64), device=device),
            torch.as_tensor(np.asarray(ids, dtype=np.int64), device=device).to(torch.uint32))


def test_known_answers(golden, cuda_device):
    ka = json.loads((golden / "known_answers.json").read_text())
    t = ka["two_element"]
    sig = signature(FeatureSet(t["ids"]), IterativeFamily(t["a"], t["b"], t["p"], t["n"]))
    assert sig.mins.tolist() == t["mins"] == [5]
    s = ka["singleton_42"]
    for kind in ("random", "iterative"):
        fam = make_family(kind, s["seed"], s["n"], s["p"])
        assert signature(FeatureSet([42]), fam).mins.tolist() == [42] * s["n"]


@pytest.mark.parametrize("out_dtype", ["int64", "uint32"])
def test_fuzz_small_primes(golden, cuda_device, out_dtype):
    z = np.load(golden / "fuzz_small.npz")
    meta = json.loads((golden / "fuzz_small.json").read_text())
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        lo, hi = z["indptr"][k], z["indptr"][k + 1]
        ip, ids = _dev([0, hi - lo], z["ids"][lo:hi], cuda_device)
        got = signatures_csr(ip, ids, fam, out_dtype=out_dtype).cpu().numpy().astype(np.int64)[0]
        assert np.array_equal(got, z["out"][z["out_ptr"][k]:z["out_ptr"][k + 1]]), m


def test_long_sets_chunk_merge(golden, cuda_device):
    z = np.load(golden / "long_sets.npz")
    meta = json.loads((golden / "long_sets.json").read_text())
    ip, ids = _dev(z["indptr"], z["ids"], cuda_device)
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        for dt in ("int64", "uint32"):
            got = signatures_csr(ip, ids, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
            assert np.array_equal(got, z[f"out{k}"]), (m, dt)


def test_cfg1_full_matches_reference_checksum(golden, cuda_device):
    meta = json.loads((golden / "cfg1.json").read_text())
    indptr, ids = gen.cfg1_numpy()
    ip, di = _dev(indptr, ids, cuda_device)
    for kind in ("random", "iterative"):
        fam = make_family(kind, meta[f"{kind}_seed"], meta["n_hash"], meta["prime"])
        out = signatures_csr(ip, di, fam, out_dtype="int64").cpu().numpy()
        assert hashlib.sha256(out.astype("<i8").tobytes()).hexdigest() == meta[f"{kind}_sha256"], kind
        out32 = signatures_csr(ip, di, fam, out_dtype="uint32").cpu().numpy()
        assert np.array_equal(out32.astype(np.int64), out)


def test_cfg1_host_pipeline(golden, cuda_device):
    """numpy in -> numpy out through mhb_sign_csr_host (the e2e entry)."""
    meta = json.loads((golden / "cfg1.json").read_text())
    indptr, ids = gen.cfg1_numpy()
    for kind in ("random", "iterative"):
        fam = make_family(kind, meta[f"{kind}_seed"], meta["n_hash"], meta["prime"])
        out = signatures_csr(indptr, ids, fam, out_dtype="int64")
        assert hashlib.sha256(out.astype("<i8").tobytes()).hexdigest() == meta[f"{kind}_sha256"], kind


@pytest.mark.parametrize("n_hash", [1, 3, 8, 17, 64, 100, 128, 255, 256, 512, 1000, 2048, 2049, 4100])
@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_lane_geometries_vs_oracle(cuda_device, n_hash, kind):
    indptr, ids = gen.cfg1_numpy(n_sets=257, seed=n_hash)
    fam = make_family(kind, 1000 + n_hash, n_hash, 1_048_583)
    ip, di = _dev(indptr, ids, cuda_device)
    got = signatures_csr(ip, di, fam).cpu().numpy()
    assert np.array_equal(got, oracle.sign_family_csr(indptr, ids, fam))


@pytest.mark.parametrize("prime", [11, 31, 101, 7757, 1_048_583, 16_777_259, 67_108_879, 1_073_741_827,
                                   1_431_655_777, 2_147_483_647])
def test_primes_up_to_2_31(cuda_device, prime):
    """Every BASELINE prime plus the narrow/wide Shoup boundary (3p vs 2^32) and 2^31-1."""
    rng = np.random.default_rng(prime)
    n_hash = min(200, (prime - 3) // 2)
    rows = [np.sort(rng.choice(prime, size=int(min(k, prime)), replace=False)) for k in rng.integers(1, 60, 64)]
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    ids = np.concatenate(rows)
    ip, di = _dev(indptr, ids, cuda_device)
    for kind in ("iterative", "random"):
        fam = make_family(kind, prime + 1, n_hash, prime)
        got = signatures_csr(ip, di, fam).cpu().numpy()
        assert np.array_equal(got, oracle.sign_family_csr(indptr, ids, fam)), kind


def test_unsorted_and_repeated_ids(cuda_device):
    """CSR rows may be unsorted and repeat ids; the result equals the canonical set's."""
    indptr, ids = gen.cfg1_numpy(n_sets=200, seed=9)
    fam = make_family("iterative", 4, 256, 1_048_583)
    want = oracle.sign_family_csr(indptr, ids, fam)
    rng = np.random.default_rng(0)
    rows = []
    for s in range(200):
        r = ids[indptr[s]:indptr[s + 1]]
        r = np.concatenate([r, r[: len(r) // 2]])
        rows.append(rng.permutation(r))
    ip2 = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    ip, di = _dev(ip2, np.concatenate(rows), cuda_device)
    assert np.array_equal(signatures_csr(ip, di, fam).cpu().numpy(), want)


def test_errors_mirror_reference(cuda_device):
    import torch

    fam = make_family("iterative", 1, 16, 7757)
    with pytest.raises(ValueError, match="empty"):
        signature(FeatureSet([]), fam)
    with pytest.raises(ValueError):
        signature(FeatureSet([5, 7757]), fam)
    ip, di = _dev([0, 2, 2, 3], [1, 2, 3], cuda_device)
    with pytest.raises(ValueError, match="empty"):
        signatures_csr(ip, di, fam)
    ip, di = _dev([0, 2], [1, 9000], cuda_device)
    with pytest.raises(ValueError):
        signatures_csr(ip, di.to(torch.uint32), fam)


def test_empty_batch(cuda_device):
    import torch

    fam = make_family("random", 1, 16, 7757)
    ip = torch.zeros(1, dtype=torch.int64, device=cuda_device)
    di = torch.zeros(0, dtype=torch.uint32, device=cuda_device)
    assert signatures_csr(ip, di, fam).shape == (0, 16)


def test_signatures_list_api(cuda_device):
    rng = np.random.default_rng(3)
    sets = [FeatureSet(rng.choice(7757, size=int(k), replace=False)) for k in rng.integers(1, 40, 50)]
    for kind in ("random", "iterative"):
        fam = make_family(kind, 8, 333, 7757)
        got = signatures(sets, fam)
        for s, g in zip(sets, got):
            assert g.family_key == fam.key
            assert np.array_equal(g.mins, oracle.brute_force_row(s.ids, fam))


def test_jaccard_estimates(golden, cuda_device):
    import torch

    z = np.load(golden / "jaccard.npz")
    meta = json.loads((golden / "jaccard.json").read_text())
    ip, di = _dev(z["indptr"], z["ids"], cuda_device)
    for fm in meta["families"]:
        fam = make_family(fm["kind"], fm["seed"], fm["n"], fm["p"])
        for dt in ("int64", "uint32"):
            sig = signatures_csr(ip, di, fam, out_dtype=dt)
            n_pairs = sig.shape[0] // 2
            pi = torch.arange(0, 2 * n_pairs, 2, device=cuda_device)
            counts, est = estimate_pairs(sig, pi, pi + 1)
            assert est.cpu().tolist() == meta["estimates"][fm["kind"]]
            blk = jaccard_block(sig[0::2].contiguous(), sig[1::2].contiguous()).cpu().numpy()
            assert np.array_equal(np.diag(blk), counts.cpu().numpy().astype(np.uint32))
            host = sig.cpu().numpy().astype(np.int64)
            want = (host[0::2][:, None, :] == host[1::2][None, :, :]).sum(-1)
            assert np.array_equal(blk.astype(np.int64), want)
        s1 = signatures([FeatureSet(z["ids"][z["indptr"][0]:z["indptr"][1]])], fam)[0]
        assert estimate_jaccard(s1, s1) == 1.0


def test_bucket_histogram(golden, cuda_device):
    for case in json.loads((golden / "hist.json").read_text()):
        fam = make_family(case["kind"], case["seed"], case["hashes"], case["prime"])
        got = bucket_histogram(case["xs"], fam, case["buckets"]).cpu().numpy()
        assert got.tolist() == case["counts"], case["kind"]


def test_cfg2_subsample_vs_oracle(cuda_device):
    """cfg2 distributions (lognormal sizes, Zipf ids over 2^24) at 20k sets vs the oracle."""
    cfg = gen.CONFIGS["cfg2"]
    ip, di = gen.make_csr(cfg, device=cuda_device, n_sets=20_000)
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    got = signatures_csr(ip, di, fam, out_dtype="uint32").cpu().numpy().astype(np.int64)
    indptr, ids = ip.cpu().numpy(), di.cpu().numpy()
    assert np.array_equal(got, oracle.sign_family_csr(indptr, ids, fam))


def test_host_pipeline_chunked_cfg2(cuda_device):
    """Host entry on a batch large enough to be cut into several chunks (rebased ids)."""
    cfg = gen.CONFIGS["cfg2"]
    ip, di = gen.make_csr(cfg, device=cuda_device, n_sets=60_000)
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    dev_out = signatures_csr(ip, di, fam, out_dtype="uint32").cpu().numpy()
    host_out = signatures_csr(ip.cpu().numpy(), di.cpu().numpy().view(np.uint32), fam, out_dtype="uint32")
    assert np.array_equal(dev_out, host_out)
    k = 2000
    ip_h = ip[:k + 1].cpu().numpy()
    want = oracle.sign_family_csr(ip_h, di[:int(ip_h[-1])].cpu().numpy().view(np.uint32), fam)
    assert np.array_equal(host_out[:k].astype(np.int64), want)


def test_band_keys_match_oracle(cuda_device):
    """cfg4 layout: N=2048 as 128 bands x 16 rows; keys equal the numpy restatement."""
    indptr, ids = gen.cfg1_numpy(n_sets=300, seed=21)
    fam = make_family("iterative", 3, 2048, 1_048_583)
    ip, di = _dev(indptr, ids, cuda_device)
    for dt in ("uint32", "int64"):
        sig = signatures_csr(ip, di, fam, out_dtype=dt)
        keys = band_keys(sig, 16).cpu().numpy()
        assert keys.shape == (300, 128)
        assert np.array_equal(keys.view(np.uint64), oracle.band_keys(sig.cpu().numpy(), 16))
    # identical sets share every band; the planted-pair mutant shares some
    ip2 = np.array([0, 50, 100], dtype=np.int64)
    row = ids[:50]
    sig2 = signatures_csr(*_dev(ip2, np.concatenate([row, row]), cuda_device), fam)
    k2 = band_keys(sig2, 16).cpu().numpy()
    assert np.array_equal(k2[0], k2[1])


def _mixed_csr(seed):
    """cfg1-like short sets plus long sets that take the merged (> kChunk) path."""
    rng = np.random.default_rng(seed)
    indptr, ids = gen.cfg1_numpy(n_sets=200, seed=seed)
    rows = [ids[indptr[s]:indptr[s + 1]] for s in range(200)]
    for n in (1025, 1500, 4096, 9000):
        rows.insert(int(rng.integers(0, len(rows))), rng.choice(1 << 20, size=n, replace=False).astype(np.uint32))
    ip = np.zeros(len(rows) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([r.size for r in rows])
    return ip, np.concatenate(rows).astype(np.uint32)


@pytest.mark.parametrize("n_hash,rows", [(2048, 16), (256, 8), (200, 8), (64, 32), (4096, 64), (128, 4)])
def test_fused_band_keys(cuda_device, n_hash, rows):
    """Keys fused into the signing epilogue equal the oracle's band keys of the
    oracle's signatures (short sets in the epilogue, long sets in finalize)."""
    indptr, ids = _mixed_csr(n_hash)
    fam = make_family("iterative", 11, n_hash, 1_048_583)
    want_sig = oracle.sign_family_csr(indptr, ids, fam)
    want = oracle.band_keys(want_sig, rows)
    ip, di = _dev(indptr, ids, cuda_device)
    for dt in ("uint32", "int64"):
        sig, keys = signatures_band_keys(ip, di, fam, rows, out_dtype=dt)
        assert np.array_equal(sig.cpu().numpy().astype(np.int64), want_sig)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), want)
    none, keys = signatures_band_keys(ip, di, fam, rows, write_signatures=False)
    assert none is None
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), want)
    # the ABI's fused mode that also stores the signatures (write_signatures = 1)
    import torch

    from paper_1401_6124_b200 import _lib

    lib = _lib.load()
    n_sets = ip.numel() - 1
    sig = torch.empty((n_sets, n_hash), dtype=torch.uint32, device=cuda_device)
    k2 = torch.empty((n_sets, n_hash // rows), dtype=torch.uint64, device=cuda_device)
    ws_bytes = lib.mhb_sign_workspace_bytes(n_sets, di.numel(), n_hash)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=cuda_device)
    _lib.check(lib.mhb_sign_iterative_csr_bands(ip.data_ptr(), di.data_ptr(), n_sets, di.numel(), fam.base.a,
                                                fam.base.b, fam.prime, n_hash, rows, k2.data_ptr(), sig.data_ptr(),
                                                _lib.OUT_U32, 1, None, ws.data_ptr(), ws_bytes,
                                                torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(sig.cpu().numpy().astype(np.int64), want_sig)
    assert np.array_equal(k2.cpu().numpy().view(np.uint64), want)


def test_fused_band_keys_fallbacks(cuda_device):
    """Random family / rows not dividing the lane count: unfused path, same keys."""
    indptr, ids = gen.cfg1_numpy(n_sets=100, seed=4)
    ip, di = _dev(indptr, ids, cuda_device)
    for fam, rows in ((make_family("random", 2, 256, 1_048_583), 16),
                      (make_family("iterative", 2, 240, 1_048_583), 48),
                      (make_family("iterative", 2, 24, 1_048_583), 4)):
        sig, keys = signatures_band_keys(ip, di, fam, rows)
        want = oracle.band_keys(oracle.sign_family_csr(indptr, ids, fam), rows)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), want)
    with pytest.raises(ValueError):
        signatures_band_keys(ip, di, make_family("iterative", 2, 256, 1_048_583), 24)


def test_fused_band_keys_abi_errors(cuda_device):
    import torch

    from paper_1401_6124_b200 import _lib

    lib = _lib.load()
    keys = torch.empty(64, dtype=torch.uint64, device=cuda_device)
    # rows not dividing n_hash -> INVALID; rows not dividing the lane count -> UNSUPPORTED
    assert lib.mhb_sign_iterative_csr_bands(None, None, 0, 0, 1, 1, 101, 256, 12, keys.data_ptr(), None, 0, 1,
                                            None, None, 0, None) == 1
    assert lib.mhb_sign_iterative_csr_bands(None, None, 0, 0, 1, 1, 101, 256, 128, keys.data_ptr(), None, 0, 1,
                                            None, None, 0, None) == 3
    assert b"rows_per_band" in lib.mhb_last_error()


@pytest.mark.parametrize("fmt", ["binary", "text"])
def test_signature_files_from_gpu(tmp_path, cuda_device, fmt):
    """GPU-formatted record files are byte-identical to the reference-format writers."""
    from paper_1401_6124_b200 import write_signatures_binary, write_signatures_text
    from paper_1401_6124_b200.records import write_signatures_csr

    indptr, ids = gen.cfg1_numpy(n_sets=777, seed=4)
    for kind, n in (("iterative", 128), ("random", 37)):
        fam = make_family(kind, 12, n, 1_048_583)
        mins = oracle.sign_family_csr(indptr, ids, fam)
        obj = np.arange(777, dtype=np.int64) * 3 + (5 if fmt == "binary" else -5)  # text allows negative ids
        ref = tmp_path / f"ref.{fmt}"
        (write_signatures_binary if fmt == "binary" else write_signatures_text)(ref, zip(obj.tolist(), mins))
        got = tmp_path / f"gpu.{fmt}"
        assert write_signatures_csr(got, indptr, ids, fam, fmt=fmt, obj_ids=obj, chunk_bytes=64 << 10) == 777
        assert got.read_bytes() == ref.read_bytes(), (kind, fmt)


@pytest.mark.parametrize("n_hash", [37, 512])
@pytest.mark.parametrize("dt", ["uint32", "int64"])
def test_pair_counts_vector_and_scalar_paths(cuda_device, n_hash, dt):
    import torch

    indptr, ids = gen.cfg1_numpy(n_sets=400, seed=n_hash)
    fam = make_family("iterative", 2, n_hash, 1_048_583)
    sig = signatures_csr(*_dev(indptr, ids, cuda_device), fam, out_dtype=dt)
    rng = np.random.default_rng(1)
    pi = rng.integers(0, 400, 1000)
    pj = rng.integers(0, 400, 1000)
    counts, est = estimate_pairs(sig, torch.as_tensor(pi, device=cuda_device), torch.as_tensor(pj, device=cuda_device))
    host = sig.cpu().numpy().astype(np.int64)
    want = (host[pi] == host[pj]).sum(1)
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), want)
    assert est.cpu().tolist() == [float(np.mean(host[a] == host[b])) for a, b in zip(pi, pj)]


def test_wide_primes_match_reference(golden, cuda_device):
    """Primes 2^31 .. 2^62: the 64-bit path equals the reference's outputs."""
    z = np.load(golden / "wide.npz")
    meta = json.loads((golden / "wide.json").read_text())
    ip, di = _dev(z["indptr"], z["ids"].astype(np.int64), cuda_device)
    for k, m in enumerate(meta):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        for dt in ("int64", "uint32"):
            got = signatures_csr(ip, di, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
            assert np.array_equal(got, z[f"out{k}"]), (m, dt)


def test_plain_c_consumer_of_the_abi(cuda_device):
    """tests/c/abi_smoke.c: a C program (no Python/torch) linking libmhb through include/mhb.h."""
    import shutil
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    src = root / "tests" / "c" / "abi_smoke.c"
    exe = root / "tests" / "c" / "abi_smoke"
    gcc = shutil.which("gcc")
    if gcc:
        cmd = [gcc, "-O2", str(src), f"-I{root / 'include'}", "-I/usr/local/cuda/include",
               f"-L{root / 'paper_1401_6124_b200' / 'lib'}", "-lmhb", "-L/usr/local/cuda/lib64", "-lcudart",
               f"-Wl,-rpath,{root / 'paper_1401_6124_b200' / 'lib'}", "-o", str(exe)]
        subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "abi_smoke ok" in r.stdout


def test_sign_corpus_matches_reference_cli(golden, tmp_path, cuda_device):
    """Text corpus -> native ingest -> GPU signatures -> GPU-formatted records: the file
    is byte-identical to the reference CLI's `sign` output (cli.py:205-230) for both
    families and formats, including the skipped empty documents' ids."""
    from paper_1401_6124_b200.corpus import sign_corpus

    cases = json.loads((golden / "corpus.json").read_text())
    for case in cases:
        if "synth" not in case:
            continue
        path = tmp_path / "corpus.txt"
        path.write_bytes(gen.synth_text_corpus(**case["synth"]))
        for key, want in case["sign_hashes16_seed3"].items():
            fam, fmt = key.split("_")
            out = tmp_path / f"sig_{key}"
            n, prime = sign_corpus(path, out, family=fam, hashes=16, seed=3, fmt=fmt, log=None)
            assert prime == case["sign_prime"]
            assert hashlib.sha256(out.read_bytes()).hexdigest() == want, (case["synth"], key)


def test_gpu_corpus_ingest_matches_reference(golden, cuda_device):
    """Device ingest (csrc/corpus_gpu.cu) == the reference's build_corpus on the golden
    corpora (edge cases + seeded synthetic text with non-ASCII lines)."""
    from paper_1401_6124_b200.corpus import build_corpus_csr

    cases = json.loads((golden / "corpus.json").read_text())
    z = np.load(golden / "corpus.npz")
    for k, case in enumerate(cases):
        data = case["text"].encode("utf-8") if "text" in case else gen.synth_text_corpus(**case["synth"])
        c = build_corpus_csr(data, backend="gpu")
        assert list(c.vocabulary.terms) == case["terms"], k
        assert c.empty_documents == case["empty"], k
        assert np.array_equal(c.indptr, z[f"indptr{k}"]), k
        assert np.array_equal(c.ids.astype(np.int64), z[f"ids{k}"]), k


@pytest.mark.parametrize("unicode_frac,crlf", [(0.0, False), (0.02, True), (0.3, False)])
def test_gpu_corpus_ingest_equals_host_backend(tmp_path, cuda_device, unicode_frac, crlf):
    """Larger corpora: GPU and host (csrc/corpus.cpp) backends agree exactly, through a
    file (pinned read) and with the CSR exported straight to device tensors."""
    import torch

    from paper_1401_6124_b200.corpus import build_corpus_csr

    text = gen.synth_text_corpus(60000, 21, vocab=80000, unicode_frac=unicode_frac, crlf=crlf)
    path = tmp_path / "c.txt"
    path.write_bytes(text)
    h = build_corpus_csr(path, backend="host")
    g = build_corpus_csr(path, backend="gpu")
    assert g.vocabulary.terms == h.vocabulary.terms and g.empty_documents == h.empty_documents
    assert np.array_equal(g.indptr, h.indptr) and np.array_equal(g.ids, h.ids)
    d = build_corpus_csr(path, backend="gpu", on_device=True)
    assert d.indptr.is_cuda and d.ids.is_cuda
    assert np.array_equal(d.indptr.cpu().numpy(), h.indptr)
    assert np.array_equal(d.ids.cpu().numpy(), h.ids)
    # and the CSR signs like the host copy
    from paper_1401_6124_b200 import make_family, signatures_csr

    fam = make_family("iterative", 1, 64, 1_048_583)
    keep = np.flatnonzero(np.diff(h.indptr) > 0)[:2000]
    rows = [h.ids[h.indptr[r]:h.indptr[r + 1]] for r in keep]
    ip = np.zeros(len(rows) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([r.size for r in rows])
    sig = signatures_csr(torch.as_tensor(ip, device=cuda_device),
                         torch.as_tensor(np.concatenate(rows).astype(np.int64), device=cuda_device).to(torch.uint32),
                         fam)
    assert np.array_equal(sig.cpu().numpy(), oracle.sign_family_csr(ip, np.concatenate(rows), fam))


def test_sign_corpus_host_backend_matches_reference_cli(golden, tmp_path, cuda_device):
    from paper_1401_6124_b200.corpus import sign_corpus

    case = [c for c in json.loads((golden / "corpus.json").read_text()) if "synth" in c][0]
    path = tmp_path / "corpus.txt"
    path.write_bytes(gen.synth_text_corpus(**case["synth"]))
    out = tmp_path / "sig"
    sign_corpus(path, out, family="random", hashes=16, seed=3, fmt="binary", backend="host", log=None)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == case["sign_hashes16_seed3"]["random_binary"]


@pytest.mark.parametrize("seed", range(8))
def test_gpu_corpus_fuzz_against_oracle(cuda_device, seed):
    """Device ingest on seeded random text (every line-break kind, Final_Sigma contexts,
    case-expanding and non-alphanumeric code points) == the pure-Python oracle."""
    from oracle import corpus_oracle
    from paper_1401_6124_b200.corpus import build_corpus_csr

    data = corpus_oracle.fuzz_text(100 + seed, 6000 + 700 * seed)
    terms, ip, x, empty = corpus_oracle.build_corpus_bytes(data)
    c = build_corpus_csr(data, backend="gpu")
    assert list(c.vocabulary.terms) == terms and c.empty_documents == empty
    assert np.array_equal(c.indptr, ip) and np.array_equal(c.ids.astype(np.int64), x)


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_small_batch_host_path(cuda_device, kind):
    """mhb_sign_csr_host's one-launch small-batch path (<= 64 sets, <= 8192 ids per set,
    N <= 16384, p < 2^32) against the oracle, at and across its limits, both dtypes."""
    from paper_1401_6124_b200.minhash import _signatures_csr_host

    rng = np.random.default_rng(17 if kind == "iterative" else 18)
    primes = [1_048_583, 16_777_259] + ([2_147_483_659, 4_294_967_291] if kind == "iterative" else [])
    for p in primes:
        for n_hash in (1, 7, 128, 1000, 16384):
            if kind == "iterative" and n_hash * 2 + 3 >= p:
                continue
            fam = make_family(kind, int(rng.integers(1 << 30)), n_hash, p)
            for sizes in ([1], [50], [8192], [8193], [3, 1, 9, 40] * 16, [5] * 65):
                if n_hash >= 1000 and sum(sizes) > 9000 and len(sizes) > 1:
                    continue
                hi = min(p, 1 << 32)
                rows = [np.unique(rng.integers(0, hi, size=n)).astype(np.uint32) for n in sizes]
                ip = np.zeros(len(rows) + 1, dtype=np.int64)
                ip[1:] = np.cumsum([r.size for r in rows])
                ids = np.concatenate(rows)
                want = oracle.sign_family_csr(ip, ids, fam)
                for dt in ("int64", "uint32"):
                    got = _signatures_csr_host(ip, ids, fam, dt, None, None)
                    assert np.array_equal(got.astype(np.int64), want), (p, n_hash, sizes[:3], dt)


def test_small_batch_status_flags(cuda_device):
    """Empty sets, ids >= p and out-of-range random parameters raise as in the reference."""
    from paper_1401_6124_b200.minhash import _signatures_csr_host

    fam = make_family("iterative", 3, 64, 1_048_583)
    with pytest.raises(ValueError):
        _signatures_csr_host(np.array([0, 2, 2], dtype=np.int64), np.array([1, 2], dtype=np.uint32), fam, "int64",
                             None, None)
    with pytest.raises(ValueError):
        signature(FeatureSet([5, 1_048_583 + 10]), fam)
    # out-of-range random parameters (a family object would reject them): status flag from both
    # the small-batch path (1 set) and the chunked pipeline (100 sets)
    import ctypes as C

    from paper_1401_6124_b200 import _lib

    lib = _lib.load()
    a = np.array([0, 5], dtype=np.uint32)
    b = np.array([1, 2], dtype=np.uint32)
    for n_sets in (1, 100):
        ip = np.arange(0, 2 * n_sets + 1, 2, dtype=np.int64)
        x = np.tile(np.array([1, 2], dtype=np.uint32), n_sets)
        out = np.empty((n_sets, 2), dtype=np.int64)
        st = C.c_int32(0)
        rc = lib.mhb_sign_csr_host(_lib.KIND_RANDOM, ip.ctypes.data, x.ctypes.data, n_sets, x.size, 0, 0,
                                   a.ctypes.data, b.ctypes.data, 1_048_583, 2, out.ctypes.data, _lib.OUT_I64,
                                   C.addressof(st), 0)
        assert rc == 0 and st.value & _lib.STATUS_BAD_PARAM, (n_sets, st.value)


def _random_unicode_text(seed, n_chars):
    """Random code points from every plane (no surrogates) mixed with ASCII words,
    separators and line breaks."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_chars):
        r = rng.random()
        if r < 0.45:
            out.append(chr(int(rng.integers(0x61, 0x7B))) if rng.random() < 0.7 else chr(int(rng.integers(0x41, 0x5B))))
        elif r < 0.6:
            out.append(" \t.,'-_"[int(rng.integers(0, 7))])
        elif r < 0.63:
            out.append(["\n", "\r\n", "\r"][int(rng.integers(0, 3))])
        else:
            while True:
                c = int(rng.integers(0x80, 0x110000)) if rng.random() < 0.3 else int(rng.integers(0x80, 0x3000))
                if not 0xD800 <= c <= 0xDFFF:
                    break
            out.append(chr(c))
    return "".join(out).encode("utf-8")


@pytest.mark.parametrize("seed", range(6))
def test_gpu_corpus_unicode_on_device(cuda_device, seed):
    """Non-ASCII lines tokenized on the device (Python's own isalnum / lower tables,
    Final_Sigma included) == the pure-Python oracle; valid UTF-8 leaves nothing for
    the caller."""
    import ctypes as C

    from oracle import corpus_oracle
    from paper_1401_6124_b200 import _lib
    from paper_1401_6124_b200.corpus import build_corpus_csr, unicode_tables

    data = _random_unicode_text(seed, 20000 + 5000 * seed)
    terms, ip, x, empty = corpus_oracle.build_corpus_bytes(data)
    c = build_corpus_csr(data, backend="gpu")
    assert list(c.vocabulary.terms) == terms and c.empty_documents == empty
    assert np.array_equal(c.indptr, ip) and np.array_equal(c.ids.astype(np.int64), x)
    # nothing goes back to Python for valid UTF-8
    lib = _lib.load()
    buf = np.frombuffer(data, dtype=np.uint8)
    h = C.c_void_p()
    _lib.check(lib.mhb_corpus_scan_device(buf.ctypes.data, buf.size, 0, C.byref(unicode_tables()), C.byref(h)))
    try:
        nd, nf = C.c_int64(), C.c_int64()
        lib.mhb_corpus_info(h, C.byref(nd), C.byref(nf))
        assert nf.value == 0
    finally:
        lib.mhb_corpus_free(h)


def test_gpu_corpus_invalid_utf8_raises(cuda_device):
    from paper_1401_6124_b200.corpus import build_corpus_csr

    for bad in (b"ok line\nbad \xc3\x28 x\n", b"a\xed\xa0\x80b\n", b"\xf4\x90\x80\x80\n", b"x\xe2\x82\n",
                b"\xc0\xaf overlong\n"):
        with pytest.raises(UnicodeDecodeError):
            build_corpus_csr(bad, backend="gpu")


def test_gpu_corpus_final_sigma(cuda_device):
    """U+03A3 in every Final_Sigma context str.lower() distinguishes: cased / uncased
    neighbours, case-ignorable runs (' . : ^ ` U+0301 U+00AD) on either side, line
    start / end, CRLF -- device ingest == the pure-Python oracle."""
    from oracle import corpus_oracle
    from paper_1401_6124_b200.corpus import build_corpus_csr

    ctx = ["", "A", "α", "1", " ", "'", ".", ":", "^", "`", "\u0301", "\u00ad", "A'", "A.", "1'", "ΑΒ", "_", "\u2019"]
    lines = []
    for left in ctx:
        for right in ctx:
            lines.append(f"{left}Σ{right}")
            lines.append(f"x {left}ΣΣ{right} y")
    data = ("\n".join(lines) + "\r\nΣ\rΑΣ").encode("utf-8")
    terms, ip, x, empty = corpus_oracle.build_corpus_bytes(data)
    c = build_corpus_csr(data, backend="gpu")
    assert list(c.vocabulary.terms) == terms and c.empty_documents == empty
    assert np.array_equal(c.indptr, ip) and np.array_equal(c.ids.astype(np.int64), x)


def test_wide_ids_beyond_2_32(golden, cuda_device):
    """The reference's int64 feature ids beyond 2^32 (primes >= 2^32): device tensors,
    numpy batches and the per-set API all equal the reference (mhb_sign_csr_ids64)."""
    import torch

    z = np.load(golden / "wide_ids.npz")
    for k, m in enumerate(json.loads((golden / "wide_ids.json").read_text())):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        ip, ids, want = z[f"indptr{k}"], z[f"ids{k}"], z[f"out{k}"]
        dev = signatures_csr(torch.as_tensor(ip, device=cuda_device), torch.as_tensor(ids, device=cuda_device), fam)
        assert np.array_equal(dev.cpu().numpy(), want), m
        assert np.array_equal(signatures_csr(ip, ids, fam), want), m
        for s in range(ip.size - 1):
            assert np.array_equal(signature(FeatureSet(ids[ip[s]:ip[s + 1]]), fam).mins, want[s]), m
        with pytest.raises(ValueError, match="int64"):
            signatures_csr(ip, ids, fam, out_dtype="uint32")


def test_random_wide_prime_host_arrays(cuda_device):
    """numpy batches with a random family over a prime >= 2^31 (64-bit a, b) run on the device."""
    rng = np.random.default_rng(8)
    fam = make_family("random", 5, 24, 3_000_000_019)
    rows = [np.unique(rng.integers(0, 2**31, size=m)) for m in (1, 9, 30)]
    ip = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int64)
    ids = np.concatenate(rows)
    got = signatures_csr(ip, ids, fam)
    for s, r in enumerate(rows):
        assert np.array_equal(got[s], oracle.brute_force_row(r, fam))


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_extreme_sets(cuda_device, kind):
    """A 5M-id set (about 4,900 merged chunks through red.global.min + finalize), a set
    of one id repeated 3000 times, ids 0 and p-1, next to ordinary sets."""
    import torch

    p = 16_777_259
    fam = make_family(kind, 9, 64, p)
    rng = np.random.default_rng(3)
    rows = [rng.integers(0, p, size=5_000_000).astype(np.uint32),  # repeats allowed: still a set
            np.full(3000, 12345, dtype=np.uint32),
            np.array([0, p - 1], dtype=np.uint32),
            np.array([p - 1], dtype=np.uint32),
            rng.integers(0, p, size=300).astype(np.uint32)]
    ip = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int64)
    ids = np.concatenate(rows)
    want = oracle.sign_family_csr(ip, ids, fam)
    got = signatures_csr(torch.as_tensor(ip, device=cuda_device),
                         torch.as_tensor(ids.astype(np.int64), device=cuda_device).to(torch.uint32), fam)
    assert np.array_equal(got.cpu().numpy(), want)
    assert np.array_equal(signatures_csr(ip, ids, fam), want)  # host pipeline, chunked


def test_signatures_list_api_ids_beyond_2_32(golden, cuda_device):
    """signatures() once narrowed int64 ids to uint32 without a check, so ids
    >= 2^32 (primes >= 2^32) were signed as different ids.  Now they reach the 64-bit-id
    path and equal the reference's outputs."""
    z = np.load(golden / "wide_ids.npz")
    for k, m in enumerate(json.loads((golden / "wide_ids.json").read_text())):
        fam = make_family(m["kind"], m["seed"], m["n"], m["p"])
        ip, ids, want = z[f"indptr{k}"], z[f"ids{k}"], z[f"out{k}"]
        if int(ids.max()) <= 2**32 - 1:
            continue
        sets = [FeatureSet(ids[ip[s]:ip[s + 1]]) for s in range(ip.size - 1)]
        got = signatures(sets, fam)
        assert all(np.array_equal(g.mins, want[s]) for s, g in enumerate(got)), m


def test_indptr_validation(cuda_device):
    """ids are read at the absolute offsets indptr[s]; indptr must start at
    >= 0, end at <= nnz and never decrease -- host and device batches both reject the rest
    before any launch."""
    import torch

    fam = make_family("iterative", 2, 64, 1_048_583)
    ids = np.arange(10, dtype=np.uint32)
    bad = [np.array([1, 5, 12], dtype=np.int64),   # ends past nnz (reads past the end from a nonzero start)
           np.array([-1, 5, 10], dtype=np.int64),  # negative start
           np.array([0, 6, 4, 10], dtype=np.int64)]  # decreasing
    for ip in bad:
        with pytest.raises(ValueError):
            signatures_csr(ip, ids, fam)
        with pytest.raises(ValueError):
            signatures_csr(torch.as_tensor(ip, device=cuda_device), torch.as_tensor(ids.astype(np.int64),
                           device=cuda_device).to(torch.uint32), fam)
    # a nonzero start that stays inside ids is fine (the ABI addresses ids[indptr[s]..])
    ip = np.array([2, 5, 10], dtype=np.int64)
    want = oracle.sign_family_csr(np.array([0, 3, 8]), ids[2:], fam)
    assert np.array_equal(signatures_csr(ip, ids, fam), want)


def test_sign_csr_device_on_a_side_stream(cuda_device):
    """the workspace belongs to the launch stream, so signing on a side stream
    while the current stream allocates and frees is safe (bit-exact, many rounds)."""
    import torch

    from paper_1401_6124_b200.minhash import sign_csr_device

    indptr, ids = gen.cfg1_numpy(n_sets=2000, seed=31)
    fam = make_family("iterative", 4, 128, 1_048_583)
    want = oracle.sign_family_csr(indptr, ids, fam)
    ip, di = _dev(indptr, ids, cuda_device)
    side = torch.cuda.Stream(cuda_device)
    outs = []
    for _ in range(20):
        out = torch.empty((indptr.size - 1, 128), dtype=torch.uint32, device=cuda_device)
        side.wait_stream(torch.cuda.current_stream())
        sign_csr_device(ip, di, fam, out, stream=side)
        junk = torch.randint(0, 1 << 30, (1 << 20,), device=cuda_device)  # current-stream churn
        del junk
        out.record_stream(side)
        outs.append(out)
    torch.cuda.synchronize()
    for out in outs:
        assert np.array_equal(out.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("kind,n_hash,p", [("iterative", 2048, 67_108_879), ("iterative", 4096, 67_108_879),
                                           ("random", 512, 4_194_319), ("random", 1000, 8_388_593)])
def test_one_set_per_warp_staged_kernel(cuda_device, kind, n_hash, p):
    """One set per warp (iterative N >= 2048; float-quotient random lanes, N >= 512) in a
    batch above the small-batch limit: the kernel stages each set's ids in shared memory
    (sets up to 133 ids), walks larger ones from global memory, and merges long sets'
    chunks -- every row against the oracle, both dtypes."""
    rng = np.random.default_rng(n_hash)
    sizes = list(rng.integers(1, 12, 17_000)) + [1, 2, 3, 117, 130, 131, 132, 133, 134, 135, 200, 257, 1024, 1025,
                                                  3000, 80, 81]
    rng.shuffle(sizes)
    rows = [np.unique(rng.integers(0, p, size=int(n))) for n in sizes]
    ip = np.zeros(len(rows) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([r.size for r in rows])
    ids = np.concatenate(rows).astype(np.uint32)
    fam = make_family(kind, 99 + n_hash, n_hash, p)
    want = oracle.sign_family_csr(ip, ids, fam)
    dip, dids = _dev(ip, ids, cuda_device)
    for dt in ("uint32", "int64"):
        got = signatures_csr(dip, dids, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, want), dt
