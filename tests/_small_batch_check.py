"""Worker for tests/test_gpu_small_batch.py: device batches of <= 16,384 sets (the
one-launch plan + sign_small_batch_kernel) against the CPU oracle, under whatever
MHB_SIGN_K / MHB_SMALL_Q the parent set (both are read once per process).

Covers: both families, both output dtypes, ragged sets from 1 id to several 1,024-id
chunks (long sets merge with red.global.min and are inverted by the last CTA), batches
of 1 set up to the small-plan limit, and the status flags (empty set, id >= p)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from paper_1401_6124_b200 import make_family, signatures_csr  # noqa: E402


def _batch(rng, sizes, hi):
    rows = [np.unique(rng.integers(0, hi, size=n)) for n in sizes]
    rows = [r if r.size else np.array([0]) for r in rows]
    ip = np.zeros(len(rows) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([r.size for r in rows])
    return ip, np.concatenate(rows).astype(np.uint32)


def main():
    import torch

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
    p = 1_048_583
    cases = [
        [1],
        [50],
        [3, 1, 9, 40] * 5,
        list(rng.poisson(50, 2000).clip(1)),
        list(rng.poisson(12, 16384).clip(1)),
        [1500, 2, 3000, 7] + list(rng.poisson(30, 300).clip(1)),  # long sets: several chunks
        [4100] * 3,
    ]
    n_checked = 0
    for kind in ("iterative", "random"):
        for n_hash in (1, 16, 128, 200, 5000):  # 5000: several lane passes (n_super > 1)
            fam = make_family(kind, int(rng.integers(1 << 30)), n_hash, p)
            for sizes in (cases if n_hash <= 200 else cases[:4] + cases[5:6]):
                ip, ids = _batch(rng, sizes, p)
                want = oracle.sign_family_csr(ip, ids, fam)
                dip = torch.as_tensor(ip, device=dev)
                dids = torch.as_tensor(ids.astype(np.int64), device=dev).to(torch.uint32)
                for dt in ("int64", "uint32"):
                    got = signatures_csr(dip, dids, fam, out_dtype=dt).cpu().numpy().astype(np.int64)
                    if not np.array_equal(got, want):
                        bad = np.argwhere(got != want)
                        raise SystemExit(f"MISMATCH {kind} N={n_hash} sets={len(sizes)} {dt}: {len(bad)} entries, "
                                         f"first {bad[:3].tolist()}")
                    n_checked += got.size
    # status flags through the device path
    fam = make_family("iterative", 11, 128, p)
    for ip, ids in ((np.array([0, 2, 2, 3], dtype=np.int64), np.array([1, 2, 3], dtype=np.uint32)),
                    (np.array([0, 2, 3], dtype=np.int64), np.array([1, p + 5, 3], dtype=np.uint32))):
        try:
            signatures_csr(torch.as_tensor(ip, device=dev),
                           torch.as_tensor(ids.astype(np.int64), device=dev).to(torch.uint32), fam)
        except ValueError:
            pass
        else:
            raise SystemExit("MISSING ValueError for an empty set / id >= p")
    # a clean call right after the failing ones reports no stale flag
    ip, ids = _batch(rng, [5, 6, 7], p)
    got = signatures_csr(torch.as_tensor(ip, device=dev),
                         torch.as_tensor(ids.astype(np.int64), device=dev).to(torch.uint32), fam).cpu().numpy()
    assert np.array_equal(got, oracle.sign_family_csr(ip, ids, fam))
    print(f"OK {n_checked} entries")


if __name__ == "__main__":
    main()
