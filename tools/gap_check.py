"""A/B of the output-sensitive iterative kernel (csrc/gap.cu, MHB_GAP=1) against the
visiting kernel (MHB_GAP=0): bit equality of the whole matrix, sampled rows against the
CPU oracle, and device time per step.  Usage: python tools/gap_check.py cfg4 [n_sets]"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1401_6124_b200 import gen, make_family  # noqa: E402
from paper_1401_6124_b200.minhash import sign_csr_device  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    cfg = gen.CONFIGS[name]
    n_sets = int(sys.argv[2]) if len(sys.argv) > 2 else min(cfg.n_sets, 2_000_000)
    n_hash = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.n_hash
    dev = torch.device("cuda", 0)
    if name == "cfg3":
        indptr, ids = gen.planted_pairs(cfg, dev, n_base=n_sets // 2)[:2]
    else:
        indptr, ids = gen.make_csr(cfg, dev, n_sets=n_sets)
    n_sets = indptr.numel() - 1
    fam = make_family("iterative", cfg.family_seed("iterative"), n_hash, cfg.prime)
    res = {"config": name, "n_sets": n_sets, "nnz": int(ids.numel()), "n_hash": n_hash, "prime": cfg.prime}
    outs = {}
    for mode in ("0", "1"):
        os.environ["MHB_GAP"] = mode
        out = torch.zeros((n_sets, n_hash), dtype=torch.uint32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        ms = timed(lambda: sign_csr_device(indptr, ids, fam, out, status))
        res["ms_gap" if mode == "1" else "ms_visit"] = ms
        res["status_" + mode] = int(status.item())
        outs[mode] = out
    res["equal"] = bool(torch.equal(outs["0"].view(torch.int32), outs["1"].view(torch.int32)))
    if not res["equal"]:
        diff = (outs["0"].view(torch.int32) != outs["1"].view(torch.int32))
        res["mismatches"] = int(diff.sum())
        r, c = torch.nonzero(diff)[0].tolist()
        res["first"] = [r, c, int(outs["0"].view(torch.int32)[r, c]), int(outs["1"].view(torch.int32)[r, c])]
    k = min(300, n_sets)
    ip = indptr[:k + 1].cpu().numpy()
    want = oracle.sign_family_csr(ip, ids[:int(ip[-1])].cpu().numpy(), fam)
    res["oracle_rows_equal"] = bool(np.array_equal(outs["1"][:k].cpu().numpy().astype(np.int64), want))
    res["speedup"] = res["ms_visit"] / res["ms_gap"]
    res["entries_per_s_gap"] = n_sets * n_hash / (res["ms_gap"] / 1e3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
