"""Seeded synthetic CSR workloads for the BASELINE configurations.

The reference measures on synthetic sets only (corpus.py:114-130);
BASELINE.json names five shapes.  These generators reproduce those shapes:

  cfg1  10,000 sets, max(1, Poisson(50)) distinct ids uniform in [0, 2^20), N=128
  cfg2  1,000,000 sets, round(lognormal(ln 120, 1.0)) clipped [1, 20000],
        Zipf(s=1.1) ids over 2^24, duplicates redrawn until the target size, N=256
  cfg3  200,000 Poisson(300) base sets over 2^22 + one mutated copy each at a target
        Jaccard J ~ U[0.1, 0.95], N=512 (planted near-duplicates; see planted_pairs)
  cfg4  2,000,000 sets, max(1, Poisson(80)) uniform over 2^26, N=2048
  cfg5  100,000,000 sets, lognormal(ln 60, 1.2) clipped [1, 50000], Zipf(1.05) over 2^30

Definitions the reference leaves open (documented in DESIGN.md):
  * Zipf is truncated to the vocabulary [1, V] (P(rank k) ~ k^-s) and rank k maps to
    id = ((k-1) * 2654435761) mod V -- an odd-multiplier bijection on [0, V) for V a
    power of two, so popular terms are scattered over the id space.
  * Sets are canonical like FeatureSet (sorted, no repeats): a repeated draw is
    redrawn until the set reaches its target size.

Two implementations: ``cfg1_numpy`` (numpy PCG64; byte-identical wherever numpy 2.3
runs -- the golden fixtures use it) and ``make_csr`` (torch; runs on the GPU for
the full-size configurations).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .families import derive_seed
from .modmath import choose_prime

MASTER_SEED = 20260810  # the reference's acceptance master seed (tests/test_acceptance.py:20)
ZIPF_SCRAMBLE = 2654435761


@dataclass(frozen=True)
class Config:
    name: str
    n_sets: int
    n_hash: int
    vocab_log2: int
    size_kind: str          # "poisson" | "lognormal"
    size_a: float           # poisson mean | lognormal median
    size_b: float           # unused | lognormal sigma
    size_cap: int           # upper clip (lognormal)
    id_kind: str            # "uniform" | "zipf"
    zipf_s: float
    families: tuple

    @property
    def vocab(self) -> int:
        return 1 << self.vocab_log2

    @property
    def prime(self) -> int:
        # choose_prime(max_id = V-1, N) (reference bench.py:66-70), fixed per config
        return choose_prime(self.vocab - 1, self.n_hash)

    def family_seed(self, kind: str) -> int:
        return derive_seed(MASTER_SEED, int(self.name[-1]), 0 if kind == "random" else 1)

    def data_seed(self) -> int:
        return derive_seed(MASTER_SEED, int(self.name[-1]), 100)


CONFIGS = {
    "cfg1": Config("cfg1", 10_000, 128, 20, "poisson", 50.0, 0.0, 1 << 62, "uniform", 0.0,
                   ("random", "iterative")),
    "cfg2": Config("cfg2", 1_000_000, 256, 24, "lognormal", 120.0, 1.0, 20_000, "zipf", 1.1, ("iterative",)),
    "cfg3": Config("cfg3", 200_000, 512, 22, "poisson", 300.0, 0.0, 1 << 62, "uniform", 0.0,
                   ("random", "iterative")),
    "cfg4": Config("cfg4", 2_000_000, 2048, 26, "poisson", 80.0, 0.0, 1 << 62, "uniform", 0.0, ("iterative",)),
    "cfg5": Config("cfg5", 100_000_000, 256, 30, "lognormal", 60.0, 1.2, 50_000, "zipf", 1.05, ("iterative",)),
}


# ---------------------------------------------------------------------------
# numpy: cfg1-shaped sets, reproducible bit for bit across machines
# ---------------------------------------------------------------------------

def cfg1_numpy(n_sets: int = 10_000, seed: int | None = None, mean: float = 50.0,
               vocab: int = 1 << 20) -> tuple[np.ndarray, np.ndarray]:
    """max(1, Poisson(mean)) distinct uniform ids per set, sorted; returns (indptr, ids uint32)."""
    rng = np.random.default_rng(CONFIGS["cfg1"].data_seed() if seed is None else seed)
    sizes = np.maximum(1, rng.poisson(mean, size=n_sets)).astype(np.int64)
    rows = [np.sort(rng.choice(vocab, size=int(k), replace=False)) for k in sizes]
    indptr = np.zeros(n_sets + 1, dtype=np.int64)
    np.cumsum(sizes, out=indptr[1:])
    ids = np.concatenate(rows).astype(np.uint32) if rows else np.zeros(0, np.uint32)
    return indptr, ids


def synth_corpus_numpy(n_docs: int, doc_size: int, seed: int, id_space: int | None = None):
    """The reference's synthetic timing corpus as CSR (restates corpus.synth_corpus,
    corpus.py:114-130): sizes uniform in [round(0.8 s), round(1.2 s)], distinct ids drawn
    with Generator.choice over id_space = max(1024, n_docs*doc_size//5), sorted like
    FeatureSet.  The same numpy calls in the same order, so the sets are identical."""
    if n_docs < 1 or doc_size < 1:
        raise ValueError("need positive document count and size")
    if id_space is None:
        id_space = max(1024, n_docs * doc_size // 5)
    lo = max(1, round(0.8 * doc_size))
    hi = max(lo, round(1.2 * doc_size))
    if id_space < hi:
        raise ValueError(f"id space {id_space} too small for documents of ~{doc_size}")
    rng = np.random.default_rng(int(seed))
    rows = []
    for _ in range(n_docs):
        sz = int(rng.integers(lo, hi + 1))
        rows.append(np.sort(rng.choice(id_space, size=sz, replace=False)))
    indptr = np.zeros(n_docs + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=indptr[1:])
    return indptr, np.concatenate(rows).astype(np.uint32)


def c6_workload():
    """Acceptance criterion C6 / the paper's Table 3 timing shape (tests/test_acceptance.py:134-149):
    500 documents of ~100 ids, N = 100,000 hashes, prime = choose_prime(max id, N)."""
    indptr, ids = synth_corpus_numpy(500, 100, derive_seed(MASTER_SEED, 6, 0))
    prime = choose_prime(int(ids.max()), 100_000)
    return indptr, ids, prime, derive_seed(MASTER_SEED, 6, 1)


_TEXT_SEPS = (b" ", b" ", b" ", b"  ", b", ", b". ", b"-", b"_", b"\t", b"!? ", b" (", b") ", b"; ", b"'")
_UNICODE_WORDS = ("caf\u00e9", "CAF\u00c9", "na\u00efve", "\u00fcber", "Stra\u00dfe", "\u0130stanbul",
                  "\u212akelvin", "\u03a3\u03bf\u03c6\u03af\u03b1", "\u65e5\u672c\u8a9e", "x\u00b2y",
                  "\u0663\u0664", "\u00e9t\u00e9", "\ufb01ne", "\u1e9e", "\u0441\u043b\u043e\u0432\u043e")


def synth_text_corpus(n_lines: int, seed: int, *, words_per_line: float = 40.0, vocab: int = 200_000,
                      zipf_s: float = 1.1, unicode_frac: float = 0.0, empty_frac: float = 0.01,
                      crlf: bool = False) -> bytes:
    """Seeded one-document-per-line text for the corpus-ingest path.

    The reference ingests real text (corpus.py:67-80) and ships none, so this stands
    in: Poisson(words_per_line) words per line drawn Zipf(zipf_s) from `vocab` random
    mixed-case ASCII words (1-14 chars of [A-Za-z0-9]), joined by separators that
    include punctuation, tabs and underscores; a fraction `empty_frac` of lines is
    empty and a fraction `unicode_frac` of lines gets one non-ASCII word (accents,
    sharp s, dotted I, Kelvin sign, Greek, CJK, ligatures, superscripts, Arabic-Indic
    digits).  Vectorised numpy, assembled in chunks."""
    rng = np.random.default_rng(int(seed))
    alpha = np.frombuffer(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789", dtype=np.uint8)
    wlen = rng.integers(1, 15, size=vocab)
    wbytes = alpha[rng.integers(0, alpha.size, size=int(wlen.sum()))]
    # lowercase-heavy: most letters lowered, so case folding merges some words
    low = (wbytes >= 65) & (wbytes <= 90) & (rng.random(wbytes.size) < 0.8)
    wbytes = np.where(low, wbytes + 32, wbytes).astype(np.uint8)
    uni = [w.encode("utf-8") for w in _UNICODE_WORDS]
    seps = list(_TEXT_SEPS)
    nl = b"\r\n" if crlf else b"\n"
    # token table: [vocab words][unicode words][separators][newline]
    table = [wbytes.tobytes()] + uni + seps + [nl]
    tlen = np.concatenate([wlen, [len(u) for u in uni], [len(x) for x in seps], [len(nl)]]).astype(np.int64)
    tstart = np.zeros(tlen.size, dtype=np.int64)
    tstart[1:] = np.cumsum(tlen)[:-1]
    blob = np.frombuffer(b"".join(table), dtype=np.uint8)
    U0, S0, NL = vocab, vocab + len(uni), vocab + len(uni) + len(seps)
    k = np.arange(1, vocab + 1, dtype=np.float64)
    cdf = np.cumsum(k ** -zipf_s)
    cdf /= cdf[-1]
    out = []
    for l0 in range(0, n_lines, 1 << 16):
        nl_ = min(n_lines - l0, 1 << 16)
        nw = rng.poisson(words_per_line, size=nl_)
        nw[rng.random(nl_) < empty_frac] = 0
        tot = int(nw.sum())
        words = np.minimum(np.searchsorted(cdf, rng.random(tot)), vocab - 1)
        has_uni = (rng.random(nl_) < unicode_frac) & (nw > 0)
        first = np.zeros(nl_, dtype=np.int64)
        first[1:] = np.cumsum(nw)[:-1]
        pick = first[has_uni] + rng.integers(0, np.maximum(nw[has_uni], 1))
        words[pick] = U0 + rng.integers(0, len(uni), size=pick.size)
        sep = S0 + rng.integers(0, len(seps), size=tot)
        # per line: w0 s0 w1 s1 ... w_{n-1} NL  (an empty line is just NL)
        cnt = np.where(nw > 0, 2 * nw, 1)
        base = np.cumsum(cnt) - cnt
        tok = np.empty(int(cnt.sum()), dtype=np.int64)
        lw = np.repeat(np.arange(nl_), nw)
        j = np.arange(tot) - first[lw]
        wpos = base[lw] + 2 * j
        tok[wpos] = words
        inner = j < nw[lw] - 1
        tok[wpos[inner] + 1] = sep[inner]
        tok[base + cnt - 1] = NL
        L = tlen[tok]
        offs = np.cumsum(L) - L
        idx = np.repeat(tstart[tok] - offs, L) + np.arange(int(L.sum()))
        out.append(blob[idx].tobytes())
    return b"".join(out)


# ---------------------------------------------------------------------------
# torch: full-size workloads (GPU) with the same distributions
# ---------------------------------------------------------------------------

class _ZipfSampler:
    """Zipf(s) truncated to ranks 1..V, drawn by inverse CDF.

    Ranks <= H (H = min(V, 2^22)) come from an exact float64 CDF table.  For V > H
    the tail k in (H, V] is drawn by inverting the continuous power law
    x^-s on [H+1/2, V+1/2] (Euler-Maclaurin midpoint approximation of the discrete
    tail, relative error ~ s/(24 k^2) per rank), weighted by its approximate mass.
    """

    HEAD = 1 << 22

    def __init__(self, s: float, vocab: int, device):
        import torch

        self.s, self.vocab = float(s), int(vocab)
        self.h = min(self.vocab, self.HEAD)
        k = torch.arange(1, self.h + 1, dtype=torch.float64, device=device)
        head = torch.cumsum(k.pow(-self.s), 0)
        head_mass = float(head[-1])
        if self.vocab > self.h:
            one_m = 1.0 - self.s
            self.lo = (self.h + 0.5) ** one_m
            self.hi = (self.vocab + 0.5) ** one_m
            tail_mass = (self.hi - self.lo) / one_m
        else:
            tail_mass = 0.0
        self.p_tail = tail_mass / (head_mass + tail_mass)
        self.cdf = head / head_mass

    def sample(self, n: int, gen):
        import torch

        dev = self.cdf.device
        u = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
        rank0 = torch.searchsorted(self.cdf, u).clamp_(max=self.h - 1)
        if self.p_tail > 0:
            v = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
            in_tail = torch.rand(n, dtype=torch.float64, device=dev, generator=gen) < self.p_tail
            x = (self.lo + v * (self.hi - self.lo)).pow(1.0 / (1.0 - self.s))
            tail0 = torch.floor(x + 0.5).to(torch.int64).clamp_(self.h + 1, self.vocab) - 1
            rank0 = torch.where(in_tail, tail0, rank0)
        return (rank0 * ZIPF_SCRAMBLE) & (self.vocab - 1)


def _draw_sizes(cfg: Config, n: int, gen, device):
    import torch

    if cfg.size_kind == "poisson":
        rates = torch.full((n,), cfg.size_a, dtype=torch.float64, device=device)
        sizes = torch.poisson(rates, generator=gen).to(torch.int64)
        return sizes.clamp_(min=1, max=min(cfg.size_cap, cfg.vocab))
    z = torch.randn(n, dtype=torch.float64, device=device, generator=gen)
    sizes = torch.round(torch.exp(math.log(cfg.size_a) + cfg.size_b * z)).to(torch.int64)
    return sizes.clamp_(min=1, max=min(cfg.size_cap, cfg.vocab))


def make_csr(cfg: Config | str, device="cuda", n_sets: int | None = None, seed: int | None = None,
             max_rounds: int = 400):
    """(indptr int64[S+1], ids uint32[nnz]) on `device`; ids sorted within each set, distinct."""
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = cfg.n_sets if n_sets is None else int(n_sets)
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed((cfg.data_seed() if seed is None else int(seed)) & ((1 << 63) - 1))
    sizes = _draw_sizes(cfg, n, gen, device)
    zipf = _ZipfSampler(cfg.zipf_s, cfg.vocab, device) if cfg.id_kind == "zipf" else None

    def draw(count: int):
        if zipf is not None:
            return zipf.sample(count, gen)
        return torch.randint(0, cfg.vocab, (count,), dtype=torch.int64, device=device, generator=gen)

    set_idx = torch.arange(n, dtype=torch.int64, device=device)
    keys = (torch.repeat_interleave(set_idx, sizes) << 32) | draw(int(sizes.sum()))
    for _ in range(max_rounds):
        keys = torch.unique(keys, sorted=True)
        have = torch.bincount(keys >> 32, minlength=n)
        deficit = sizes - have
        missing = int(deficit.sum())
        if missing == 0:
            break
        extra = (torch.repeat_interleave(set_idx, deficit) << 32) | draw(missing)
        keys = torch.cat([keys, extra])
    else:
        raise RuntimeError("duplicate redraw did not converge")
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(sizes, 0, out=indptr[1:])
    ids = (keys & 0xFFFFFFFF).to(torch.uint32)
    return indptr, ids


def planted_pairs(cfg: Config | str = "cfg3", device="cuda", n_base: int | None = None, seed: int | None = None,
                  j_lo: float = 0.1, j_hi: float = 0.95, max_rounds: int = 100):
    """cfg3: base sets (Poisson(300) over 2^22) each followed by a mutated copy.

    For base set k of size n the mutant keeps c = round(2nJ/(1+J)) base ids (a
    random subset) and adds n - c fresh ids absent from the base, so the pair's
    exact Jaccard is c / (2n - c) (the construction of corpus.synth_pair,
    corpus.py:83-111, with a per-pair target J ~ U[j_lo, j_hi]).  Sets 2k and 2k+1
    form pair k, so nnz-balanced sharding with align=2 never splits a pair.
    Returns (indptr int64[2B+1], ids uint32, exact_jaccard float64[B]).
    """
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n_base = cfg.n_sets if n_base is None else int(n_base)
    device = torch.device(device)
    seed = cfg.data_seed() if seed is None else int(seed)
    b_ip, b_ids = make_csr(cfg, device=device, n_sets=n_base, seed=seed)
    gen = torch.Generator(device=device)
    gen.manual_seed((seed + 1) & ((1 << 63) - 1))
    sizes = b_ip[1:] - b_ip[:-1]
    j = j_lo + (j_hi - j_lo) * torch.rand(n_base, dtype=torch.float64, device=device, generator=gen)
    keep = torch.round(2.0 * sizes.double() * j / (1.0 + j)).to(torch.int64).clamp_(min=1)
    keep = torch.minimum(keep, sizes)
    set_idx = torch.arange(n_base, dtype=torch.int64, device=device)
    owner = torch.repeat_interleave(set_idx, sizes)
    base_keys = (owner << 32) | b_ids.to(torch.int64)
    # random subset of size keep[k] of each base set: rank elements by a random key
    r = torch.rand(owner.numel(), device=device, generator=gen)
    order = torch.argsort(owner.double() * 2.0 + r)  # stable grouping by set, random inside
    pos = torch.arange(owner.numel(), device=device) - torch.repeat_interleave(b_ip[:-1], sizes)
    kept = base_keys[order][pos < keep[owner]]
    # fresh ids: uniform over the vocabulary, not in the base set, no repeats
    need = sizes - keep
    fresh = torch.empty(0, dtype=torch.int64, device=device)
    sorted_base = torch.sort(base_keys).values
    for _ in range(max_rounds):
        have = torch.bincount(fresh >> 32, minlength=n_base) if fresh.numel() else torch.zeros_like(need)
        deficit = need - have
        missing = int(deficit.sum())
        if missing == 0:
            break
        cand = (torch.repeat_interleave(set_idx, deficit) << 32) | torch.randint(
            0, cfg.vocab, (missing,), dtype=torch.int64, device=device, generator=gen)
        pos_b = torch.searchsorted(sorted_base, cand).clamp_(max=sorted_base.numel() - 1)
        cand = cand[sorted_base[pos_b] != cand]
        fresh = torch.unique(torch.cat([fresh, cand]))
    else:
        raise RuntimeError("fresh-id redraw did not converge")
    mut_keys = torch.sort(torch.cat([kept, fresh])).values
    # interleave: base k -> set 2k, mutant k -> set 2k+1
    b_sorted = torch.sort(base_keys).values
    all_keys = torch.cat([((b_sorted >> 32) * 2) << 32 | (b_sorted & 0xFFFFFFFF),
                          ((mut_keys >> 32) * 2 + 1) << 32 | (mut_keys & 0xFFFFFFFF)])
    all_keys = torch.sort(all_keys).values
    counts = torch.bincount(all_keys >> 32, minlength=2 * n_base)
    indptr = torch.zeros(2 * n_base + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=indptr[1:])
    ids = (all_keys & 0xFFFFFFFF).to(torch.uint32)
    exact = keep.double() / (2.0 * sizes.double() - keep.double())
    return indptr, ids, exact


# ---------------------------------------------------------------------------
# Blocked batches: one global batch, any slice of it generated on its own
# ---------------------------------------------------------------------------
#
# The multi-GPU driver cuts ONE global batch into nnz-balanced row shards and every
# rank generates only its own shard on its own device.  So the batch is a sequence of
# fixed blocks of BLOCK_SETS sets (pairs for cfg3), block b drawn by make_csr /
# planted_pairs from its own seed derive_seed(data_seed, 7, b).  make_csr draws a
# block's sizes first from that seed, so every rank can rebuild the global indptr from
# the sizes alone (a few kernels per block), cut it, and generate just the blocks its
# rows touch.  The batch is identical for any world size.

BLOCK_SETS = 1 << 18


def _block_seed(seed: int, b: int) -> int:
    return derive_seed(seed, 7, b)


def _planted(cfg: Config) -> bool:
    return cfg.name == "cfg3"


def block_layout(cfg: Config | str, n_sets: int | None = None, block: int = BLOCK_SETS):
    """(unit, sets_per_block, n_blocks, n_sets): cfg3 blocks hold `block` planted pairs."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    unit = 2 if _planted(cfg) else 1
    n = (cfg.n_sets * unit if n_sets is None else int(n_sets))
    if n % unit:
        raise ValueError("planted-pair batches hold an even number of sets")
    bs = block * unit
    return unit, bs, (n + bs - 1) // bs, n


def global_sizes(cfg: Config | str, device="cuda", n_sets: int | None = None, seed: int | None = None,
                 block: int = BLOCK_SETS):
    """int64[S] set sizes of the blocked batch (no ids drawn)."""
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    device = torch.device(device)
    seed = cfg.data_seed() if seed is None else int(seed)
    unit, bs, nb, n = block_layout(cfg, n_sets, block)
    parts = []
    for b in range(nb):
        nb_sets = min(bs, n - b * bs) // unit
        g = torch.Generator(device=device)
        g.manual_seed(_block_seed(seed, b) & ((1 << 63) - 1))
        s = _draw_sizes(cfg, nb_sets, g, device)
        parts.append(torch.repeat_interleave(s, unit) if unit > 1 else s)
    return torch.cat(parts) if parts else torch.zeros(0, dtype=torch.int64, device=device)


def global_indptr(cfg: Config | str, device="cuda", n_sets: int | None = None, seed: int | None = None,
                  block: int = BLOCK_SETS):
    import torch

    sizes = global_sizes(cfg, device, n_sets, seed, block)
    ip = torch.zeros(sizes.numel() + 1, dtype=torch.int64, device=sizes.device)
    torch.cumsum(sizes, 0, out=ip[1:])
    return ip


def make_shard(cfg: Config | str, s0: int, s1: int, device="cuda", n_sets: int | None = None,
               seed: int | None = None, block: int = BLOCK_SETS, indptr=None):
    """Sets [s0, s1) of the blocked global batch on `device`.

    Returns (indptr int64[s1-s0+1] starting at 0, ids uint32, exact_jaccard or None);
    exact_jaccard (cfg3) holds the planted pairs of the slice, which must then start and
    end on a pair boundary.  `indptr`: the global indptr if the caller has it."""
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    device = torch.device(device)
    seed = cfg.data_seed() if seed is None else int(seed)
    unit, bs, nb, n = block_layout(cfg, n_sets, block)
    if not (0 <= s0 <= s1 <= n):
        raise ValueError(f"slice [{s0}, {s1}) outside the batch of {n} sets")
    if unit > 1 and (s0 % unit or s1 % unit):
        raise ValueError("planted-pair slices must start and end on a pair boundary")
    if indptr is None:
        indptr = global_indptr(cfg, device, n, seed, block)
    ip_g = indptr.to(device)
    lo = int(ip_g[s0])
    local_ip = (ip_g[s0:s1 + 1] - lo).contiguous()
    nnz = int(local_ip[-1])
    ids = torch.empty(nnz, dtype=torch.uint32, device=device)
    exact = [] if unit > 1 else None
    for b in range(s0 // bs, (s1 + bs - 1) // bs):
        b_lo, b_hi = b * bs, min(n, (b + 1) * bs)
        r0, r1 = max(s0, b_lo) - b_lo, min(s1, b_hi) - b_lo
        if r1 <= r0:
            continue
        bseed = _block_seed(seed, b)
        if unit > 1:
            bip, bids, bj = planted_pairs(cfg, device=device, n_base=(b_hi - b_lo) // 2, seed=bseed)
            exact.append(bj[r0 // 2:r1 // 2])
        else:
            bip, bids = make_csr(cfg, device=device, n_sets=b_hi - b_lo, seed=bseed)
        a, z = int(bip[r0]), int(bip[r1])
        dst = int(ip_g[b_lo + r0]) - lo
        ids[dst:dst + (z - a)].copy_(bids[a:z])
        del bip, bids
    return local_ip, ids, (torch.cat(exact) if exact is not None and exact else exact)
