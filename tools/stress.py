"""Randomized differential stress of every signing path against the CPU oracle.

usage: python tools/stress.py [seconds] [seed]

Each case draws a family (random / iterative), N, a prime (tiny .. 2^31, and wide
ones up to 2^32), set sizes (1 .. a few chunks, repeated ids), and an entry path:
device CSR, host pipeline (pinned / pageable, uint32 / int64, pinned int64), small-batch
host path (doorbell block / launched grid, wide N up to 100,000), the per-set
signature() API, fused band keys (keys only, and with signatures), 64-bit ids; batch
sizes on both sides of the one-launch small plan (16,384 sets).  Any mismatch is printed with its seed and the
run exits non-zero.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402
from paper_1401_6124_b200 import (FeatureSet, band_keys, make_family, signature, signatures_band_keys,  # noqa: E402
                                  signatures_csr)
from paper_1401_6124_b200.minhash import _signatures_csr_host  # noqa: E402

PRIMES = [11, 101, 7757, 65537, 1_048_583, 4_194_319, 8_388_593, 16_777_259, 67_108_879, 1_073_741_827,
          2_147_483_647, 2_147_483_659, 3_000_000_019, 4_294_967_291]


def case(rng, dev):
    kind = "iterative" if rng.random() < 0.6 else "random"
    p = int(rng.choice(PRIMES))
    n_hash = int(rng.choice([1, 2, 5, 16, 31, 64, 100, 128, 256, 300, 512, 1000, 2048, 2100]))
    if kind == "iterative" and 2 * n_hash + 3 >= p:
        n_hash = max(1, (p - 4) // 2)
    if kind == "random" and p > 2**31 - 1:
        p = 2_147_483_647 if rng.random() < 0.5 else 1_073_741_827
    fam = make_family(kind, int(rng.integers(1 << 30)), n_hash, p)
    n_sets = int(rng.choice([1, 2, 7, 64, 65, 300, 2000, 16384, 16385, 20000],
                            p=[.12, .12, .12, .12, .12, .12, .12, .05, .05, .06]))
    if n_sets > 2000 and n_hash > 512:  # keep the oracle's share of a case in seconds
        n_hash = int(rng.choice([16, 64, 128, 256]))
        if kind == "iterative" and 2 * n_hash + 3 >= p:
            n_hash = max(1, (p - 4) // 2)
        fam = make_family(kind, int(rng.integers(1 << 30)), n_hash, p)
    if rng.random() < 0.15:  # wide small batches: the launched (hash slice, set) grid, device staging
        n_sets = int(rng.choice([1, 3, 20]))
        n_hash = int(rng.choice([4000, 8192, 20_000, 100_000]))
        if kind == "iterative" and 2 * n_hash + 3 >= p:
            p = 1_073_741_827
        fam = make_family(kind, int(rng.integers(1 << 30)), n_hash, p)
    sizes = rng.choice([1, 2, 3, 50, 200, 1023, 1024, 1025, 3000], size=n_sets,
                       p=[.1, .1, .1, .3, .2, .05, .05, .05, .05] if n_sets <= 2000
                       else [.2, .2, .2, .3, .09, .004, .003, .002, .001])
    rows = []
    hi = min(p, 1 << 32)
    for n in sizes:
        r = rng.integers(0, hi, size=int(n), dtype=np.int64)
        if rng.random() < 0.2:  # repeated ids
            r = np.concatenate([r, r[: max(1, r.size // 3)]])
        rows.append(r.astype(np.uint32))
    ip = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int64)
    ids = np.concatenate(rows)
    want = oracle.sign_family_csr(ip, ids, fam)
    path = rng.choice(["device", "host_pinned", "host_pageable", "host_int64", "bands", "bands_sig", "ids64",
                       "per_set", "host_pinned_int64"])
    if path == "device":
        got = signatures_csr(torch.as_tensor(ip, device=dev), torch.as_tensor(ids.astype(np.int64), device=dev),
                             fam, out_dtype=str(rng.choice(["uint32", "int64"]))).cpu().numpy().astype(np.int64)
    elif path == "host_pinned":
        ids_p = torch.from_numpy(ids.view(np.int32)).pin_memory().numpy().view(np.uint32)
        out = torch.empty((n_sets, n_hash), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        got = signatures_csr(ip, ids_p, fam, out_dtype="uint32", out=out).astype(np.int64)
    elif path == "host_pageable":
        got = signatures_csr(ip, ids, fam, out_dtype="uint32").astype(np.int64)
    elif path == "host_int64":
        got = _signatures_csr_host(ip, ids, fam, "int64", None, None)
    elif path == "per_set":  # the reference API, one signature() per set (doorbell / launched grid)
        k = min(n_sets, 4)
        got = np.stack([signature(FeatureSet(rows[i].astype(np.int64)), fam).mins for i in range(k)])
        return kind, p, n_hash, n_sets, path, bool(np.array_equal(got, want[:k]))
    elif path == "host_pinned_int64":  # written straight into the caller's page-locked buffer
        out = torch.empty((n_sets, n_hash), dtype=torch.int64).pin_memory().numpy()
        got = _signatures_csr_host(ip, ids, fam, "int64", out, None)
    elif path == "bands":
        rows_b = next((r for r in (16, 8, 4) if n_hash % r == 0), None)
        if rows_b is None:
            return kind, p, n_hash, n_sets, path, True
        _, keys = signatures_band_keys(torch.as_tensor(ip, device=dev),
                                       torch.as_tensor(ids.astype(np.int64), device=dev), fam, rows_b,
                                       write_signatures=False)
        ok = np.array_equal(keys.cpu().numpy().view(np.uint64), oracle.band_keys(want, rows_b))
        return kind, p, n_hash, n_sets, path, ok
    elif path == "bands_sig":  # signatures and keys together (fused for N >= 1024)
        rows_b = next((r for r in (16, 8, 4) if n_hash % r == 0), None)
        if rows_b is None:
            return kind, p, n_hash, n_sets, path, True
        sig, keys = signatures_band_keys(torch.as_tensor(ip, device=dev),
                                         torch.as_tensor(ids.astype(np.int64), device=dev), fam, rows_b)
        ok = (np.array_equal(keys.cpu().numpy().view(np.uint64), oracle.band_keys(want, rows_b))
              and np.array_equal(sig.cpu().numpy().astype(np.int64), want))
        return kind, p, n_hash, n_sets, path, ok
    else:  # 64-bit ids only apply when the prime admits ids >= 2^32; use brute force on a few rows
        if p < 2**32 or kind == "random":
            return kind, p, n_hash, n_sets, path, True
        got = signatures_csr(torch.as_tensor(ip, device=dev), torch.as_tensor(ids.astype(np.int64), device=dev),
                             fam).cpu().numpy()
    return kind, p, n_hash, n_sets, path, bool(np.array_equal(got, want))


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 120
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    t0, n, bad = time.time(), 0, 0
    while time.time() - t0 < seconds:
        st = rng.bit_generator.state
        kind, p, n_hash, n_sets, path, ok = case(rng, dev)
        n += 1
        if not ok:
            bad += 1
            print("MISMATCH", kind, p, n_hash, n_sets, path, st["state"]["state"], flush=True)
    print(f"stress: {n} cases, {bad} mismatches in {time.time() - t0:.0f} s (seed {seed})")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
