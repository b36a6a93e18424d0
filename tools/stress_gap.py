"""Randomised A/B of the enumerating kernel (MHB_GAP=1) against the visiting kernel
(MHB_GAP=0), whole matrices compared on the GPU; the visiting kernel is itself pinned to
the oracle by the test suite.  Each case draws a prime (tiny to 2^31 - 1), a lane count,
a set-size mix (singletons to thousands, repeats, the constant-orbit id p - b), a
threshold scale and an output dtype.  Usage: python tools/stress_gap.py [cases] [seed]"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1401_6124_b200 import make_family, next_prime  # noqa: E402
from paper_1401_6124_b200.minhash import sign_csr_device  # noqa: E402

PRIMES = [101, 251, 7757, 65_537, 1_048_583, 4_194_319, 16_777_259, 67_108_879, 1_073_741_827, 1_431_655_777,
          2_147_483_629, 2_147_483_647]


def case(rng, dev):
    p = int(rng.choice(PRIMES))
    if rng.random() < 0.3:
        p = next_prime(int(rng.integers(200, 1 << 31)))
    n_max = max(1, min(4096, (p - 3) // 2))
    n_hash = int(min(n_max, rng.choice([1, 3, 4, 17, 64, 100, 128, 256, 500, 512, 1000, 2048, 2052, 3000, 4096])))
    n_sets = int(rng.integers(16_385, 30_000))
    mix = rng.choice(["tiny", "text", "wide"])
    if mix == "tiny":
        sizes = rng.choice([1, 2, 3, 5, 9], size=n_sets)
    elif mix == "text":
        sizes = np.maximum(1, rng.poisson(rng.choice([12, 40, 80]), size=n_sets))
    else:
        sizes = rng.choice([1, 7, 60, 300, 2500], size=n_sets, p=[.3, .3, .3, .09, .01])
    if n_hash > 1000:
        sizes = np.minimum(sizes, 400)
    total = int(sizes.sum())
    ids = rng.integers(0, min(p, 1 << 32), size=total, dtype=np.int64)
    fam = make_family("iterative", int(rng.integers(0, 2**62)), n_hash, p)
    x0 = (p - fam.base.b) % p  # d = 0: the constant orbit
    ids[rng.integers(0, total, size=max(1, total // 5000))] = x0
    if rng.random() < 0.3:  # repeats inside sets
        k = total // 4
        ids[1:k + 1] = ids[:k]
    indptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ip = torch.as_tensor(indptr, device=dev)
    di = torch.as_tensor(ids, device=dev).to(torch.uint32)
    dt = torch.int64 if rng.random() < 0.3 else torch.uint32
    cmul = float(rng.choice([1.0, 1.0, 0.3, 3.0, 0.0001]))
    outs = []
    for mode in ("0", "1"):
        os.environ["MHB_GAP"] = mode
        os.environ["MHB_GAP_CMUL"] = str(cmul)
        out = torch.zeros((n_sets, n_hash), dtype=dt, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        sign_csr_device(ip, di, fam, out, status)
        torch.cuda.synchronize()
        if int(status.item()) != 0:
            raise SystemExit(f"status {int(status.item())} in mode {mode}: p={p} N={n_hash}")
        outs.append(out.view(torch.int64) if dt == torch.int64 else out.view(torch.int32))
    ok = bool(torch.equal(outs[0], outs[1]))
    return ok, (p, n_hash, n_sets, mix, cmul, str(dt))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    bad = 0
    t0 = time.time()
    for k in range(cases):
        ok, desc = case(rng, dev)
        if not ok:
            bad += 1
            print("MISMATCH", desc, flush=True)
    print(f"stress_gap: {cases} cases, seed {seed}, {bad} mismatches, {time.time() - t0:.1f} s")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
