"""Strong-scaling projection of the compute phase from per-shard timings on ONE GPU.

usage: python tools/scaling_projection.py [config] [steps]      (default cfg4, 10)

For N in 1, 2, 4, 8 the global batch is cut exactly as `bench.py --gpus N` cuts it
(dist.nnz_balanced_cuts of the blocked batch's indptr); every rank's shard is generated
(gen.make_shard) and signed alone on this GPU, K steps timed with CUDA events after
warm-up.  The N-GPU compute phase takes the slowest shard's time, so

    projected value(N) = S * N_hash / max_r t_r,   efficiency(N) = value(N) / (N * value(1)).

This is a projection, not a multi-GPU measurement: it leaves out NVLink, NCCL and
per-GPU clock differences (there is no collective in the compute phase; the gathers are
reported separately by bench.py).  Prints one JSON line.
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_1401_6124_b200 import gen, make_family
    from paper_1401_6124_b200.dist import nnz_balanced_cuts
    from paper_1401_6124_b200.minhash import sign_csr_to_ptr

    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cfg = gen.CONFIGS[cfg_name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    unit, _, _, n_total = gen.block_layout(cfg)
    ip_g = gen.global_indptr(cfg, dev, n_total)
    fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
    N = cfg.n_hash
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    res = {}
    for world in (1, 2, 4, 8):
        cuts = nnz_balanced_cuts(ip_g, world, align=unit)
        times, nnzs = [], []
        for r in range(world):
            s0, s1 = cuts[r], cuts[r + 1]
            ip, ids, _ = gen.make_shard(cfg, s0, s1, dev, n_total, indptr=ip_g)
            out = torch.empty((s1 - s0, N), dtype=torch.uint32, device=dev)
            for _ in range(2):
                sign_csr_to_ptr(ip, ids, fam, out.data_ptr(), False, status, stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                sign_csr_to_ptr(ip, ids, fam, out.data_ptr(), False, status, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            if int(status.item()):
                raise SystemExit(f"status flags {int(status.item())}")
            times.append(e0.elapsed_time(e1) / steps)
            nnzs.append(int(ids.numel()))
            del out, ip, ids
            torch.cuda.empty_cache()
        t = max(times)
        res[world] = {"ms_per_step": t, "value": n_total * N / (t / 1e3),
                      "shard_ms": [round(x, 4) for x in times], "shard_nnz": nnzs, "cuts": cuts}
    v1 = res[1]["value"]
    for world, r in res.items():
        r["efficiency"] = r["value"] / (world * v1)
    print(json.dumps({"metric": "projected compute-phase entries/s (strong scaling, per-shard timings on one B200)",
                      "config": cfg_name, "n_sets": n_total, "n_hash": N, "steps": steps,
                      "method": "dist.nnz_balanced_cuts of the global batch; every rank's shard signed alone on "
                                "this GPU; value(N) = S*N / max over ranks; no NVLink / NCCL in the compute phase",
                      "gpu": torch.cuda.get_device_name(dev), "when": time.strftime("%Y-%m-%d %H:%M:%S"),
                      "by_world": res}))


if __name__ == "__main__":
    main()
