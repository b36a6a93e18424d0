"""Full BASELINE sizes (cfg2: 1M sets x 256, cfg3: 400k x 512, cfg4: 2M x 2048) through
size-independent properties (the oracle cannot run these sizes in seconds):

  * membership  -- every argmin id belongs to its own set (the signature of a set is a
                   vector of its members, minhash.py:94-96);
  * exactness   -- bit-equality with the CPU oracle on a spread sample of sets,
                   including the largest (merged) ones;
  * invariance  -- shuffling the ids inside every set changes nothing (the argmin of a
                   bijection is order-free; the reference sorts via FeatureSet);
  * paths agree -- the chunked host pipeline and the fused band-key epilogue reproduce
                   the device path / the standalone kernel at full size;
  * statistics  -- cfg3 planted pairs: estimates track the exact Jaccard.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import band_keys, estimate_pairs, gen, make_family, signatures_band_keys, signatures_csr

pytestmark = pytest.mark.gpu


def _membership(ip, ids, sig):
    """Every sig[s, i] is one of ids[ip[s]:ip[s+1]] (rows are sorted, as gen emits them)."""
    import torch

    n_sets, n_hash = sig.shape
    sizes = ip[1:] - ip[:-1]
    set_of = torch.repeat_interleave(torch.arange(n_sets, device=ids.device), sizes)
    keys = (set_of << 32) | ids.view(torch.int32).to(torch.int64)
    assert bool((keys[1:] > keys[:-1]).all()), "rows must be sorted and duplicate-free"
    step = max(1, (1 << 27) // n_hash)
    for s0 in range(0, n_sets, step):
        s1 = min(n_sets, s0 + step)
        q = (torch.arange(s0, s1, device=ids.device, dtype=torch.int64)[:, None] << 32) | sig[s0:s1].view(
            torch.int32).to(torch.int64)
        pos = torch.searchsorted(keys, q.reshape(-1)).clamp_(max=keys.numel() - 1)
        assert bool((keys[pos] == q.reshape(-1)).all()), f"an argmin outside its set in rows {s0}..{s1}"


def _sample_rows(ip, k, rng):
    """k spread rows plus the largest rows."""
    n = ip.numel() - 1
    sizes = (ip[1:] - ip[:-1]).cpu().numpy()
    pick = np.unique(np.concatenate([rng.choice(n, size=k, replace=False), np.argsort(sizes)[-8:]]))
    return pick


def _rows(sig, rows):
    import torch

    return sig.view(torch.int32)[torch.as_tensor(rows, device=sig.device)].cpu().numpy().astype(np.int64)


def _oracle_rows(ip, ids, fam, rows):
    ip_h = ip.cpu().numpy()
    parts = [ids[int(ip_h[r]):int(ip_h[r + 1])].cpu().numpy().view(np.uint32) for r in rows]
    sub_ip = np.concatenate([[0], np.cumsum([p.size for p in parts])]).astype(np.int64)
    return oracle.sign_family_csr(sub_ip, np.concatenate(parts), fam)


def _shuffled_within_sets(ip, ids, seed):
    import torch

    g = torch.Generator(device=ids.device).manual_seed(seed)
    sizes = ip[1:] - ip[:-1]
    set_of = torch.repeat_interleave(torch.arange(ip.numel() - 1, device=ids.device), sizes)
    r = torch.rand(ids.numel(), generator=g, device=ids.device)
    order = torch.argsort(set_of.double() + r.double())  # stable set blocks, random order inside
    return ids.view(torch.int32)[order].view(torch.uint32)


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_cfg2_full(cuda_device, kind):
    import torch

    cfg = gen.CONFIGS["cfg2"]
    ip, ids = gen.make_csr(cfg, device=cuda_device)
    assert ip.numel() - 1 == cfg.n_sets
    fam = make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
    sig = signatures_csr(ip, ids, fam, out_dtype="uint32")
    _membership(ip, ids, sig)
    rows = _sample_rows(ip, 3000, np.random.default_rng(1))
    assert np.array_equal(_rows(sig, rows), _oracle_rows(ip, ids, fam, rows))
    sig2 = signatures_csr(ip, _shuffled_within_sets(ip, ids, 5), fam, out_dtype="uint32")
    assert torch.equal(sig2.view(torch.int32), sig.view(torch.int32))
    if kind == "iterative":  # the host pipeline (chunked H2D / kernels / D2H) on the full batch
        host = signatures_csr(ip.cpu().numpy(), ids.cpu().numpy().view(np.uint32), fam, out_dtype="uint32")
        assert np.array_equal(host, sig.cpu().numpy())


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_cfg3_full_planted_pairs(cuda_device, kind):
    cfg = gen.CONFIGS["cfg3"]
    ip, ids, exact_j = gen.planted_pairs(cfg, device=cuda_device)
    fam = make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
    sig = signatures_csr(ip, ids, fam, out_dtype="uint32")
    _membership(ip, ids, sig)
    rows = _sample_rows(ip, 1500, np.random.default_rng(2))
    assert np.array_equal(_rows(sig, rows), _oracle_rows(ip, ids, fam, rows))
    import torch

    n_pairs = (ip.numel() - 1) // 2
    pi = torch.arange(0, 2 * n_pairs, 2, device=cuda_device)
    counts, est = estimate_pairs(sig, pi, pi + 1)
    err = (est - exact_j).abs()
    assert float(err.mean()) < 0.03  # N=512: sd of one estimate <= 0.022
    assert float(err.max()) < 0.25


def test_cfg4_full_with_fused_band_keys(cuda_device):
    import torch

    cfg = gen.CONFIGS["cfg4"]
    ip, ids = gen.make_csr(cfg, device=cuda_device)
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    sig, keys = signatures_band_keys(ip, ids, fam, 16)
    _membership(ip, ids, sig)
    rows = _sample_rows(ip, 600, np.random.default_rng(3))
    assert np.array_equal(_rows(sig, rows), _oracle_rows(ip, ids, fam, rows))
    assert torch.equal(keys.view(torch.int64), band_keys(sig, 16).view(torch.int64))
    _, keys_only = signatures_band_keys(ip, ids, fam, 16, write_signatures=False)
    assert torch.equal(keys_only.view(torch.int64), keys.view(torch.int64))


def _zipf_sets(cfg, sizes, device, seed):
    """Distinct Zipf(cfg) ids over cfg's vocabulary for sets of the given sizes (sorted)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    z = gen._ZipfSampler(cfg.zipf_s, cfg.vocab, device)
    rows = []
    for n in sizes:
        have = torch.empty(0, dtype=torch.int64, device=device)
        while have.numel() < n:
            have = torch.unique(torch.cat([have, z.sample(4 * n, g)]))
        # keep n distinct ids: a random subset, so popular and rare ids both appear
        keep = have[torch.randperm(have.numel(), generator=g, device=device)[:n]]
        rows.append(torch.sort(keep).values.to(torch.uint32))
    return rows


def test_cfg5_distribution_shard(cuda_device):
    """cfg5's generator (lognormal(60, 1.2) sizes, Zipf(1.05) ids over 2^30, p =
    1,073,741,827: the largest BASELINE prime, 3p < 2^32) on its first 200k sets plus
    sets at the 50,000-id cap: membership, oracle rows (including the capped sets, which
    merge 49 chunks each), shuffle invariance, and the host pipeline."""
    import torch

    cfg = gen.CONFIGS["cfg5"]
    ip0, ids0, _ = gen.make_shard(cfg, 0, 200_000, cuda_device)
    big = _zipf_sets(cfg, [50_000, 50_000, 49_999, 20_001], cuda_device, 7)
    ids = torch.cat([ids0] + big)
    sizes = torch.cat([ip0[1:] - ip0[:-1], torch.tensor([b.numel() for b in big], device=cuda_device)])
    ip = torch.zeros(sizes.numel() + 1, dtype=torch.int64, device=cuda_device)
    torch.cumsum(sizes, 0, out=ip[1:])
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    assert fam.prime == 1_073_741_827
    sig = signatures_csr(ip, ids, fam, out_dtype="uint32")
    _membership(ip, ids, sig)
    n = ip.numel() - 1
    rows = np.unique(np.concatenate([_sample_rows(ip, 2000, np.random.default_rng(4)), np.arange(n - 4, n)]))
    assert np.array_equal(_rows(sig, rows), _oracle_rows(ip, ids, fam, rows))
    sig2 = signatures_csr(ip, _shuffled_within_sets(ip, ids, 9), fam, out_dtype="uint32")
    assert torch.equal(sig2.view(torch.int32), sig.view(torch.int32))
    host = signatures_csr(ip.cpu().numpy(), ids.cpu().numpy().view(np.uint32), fam, out_dtype="int64")
    assert np.array_equal(host, sig.cpu().numpy().astype(np.int64))
