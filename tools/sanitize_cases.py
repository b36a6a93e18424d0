"""Small runs of every libmhb path, for `compute-sanitizer --tool memcheck` on the box."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1401_6124_b200 import bucket_histogram, estimate_pairs, gen, jaccard_block, make_family, signatures_csr  # noqa: E402

dev = torch.device("cuda", 0)
cfg = gen.CONFIGS["cfg2"]
ip, ids = gen.make_csr(cfg, device=dev, n_sets=30_000)          # lognormal sizes, long sets, Zipf ids
ip_h, ids_h = ip.cpu().numpy(), ids.cpu().numpy().view(np.uint32)
for kind in ("iterative", "random"):
    for n_hash in (7, 100, 256, 2100):
        fam = make_family(kind, 5, n_hash, cfg.prime)
        for dt in ("uint32", "int64"):
            d = signatures_csr(ip, ids, fam, out_dtype=dt)
            h = signatures_csr(ip_h, ids_h, fam, out_dtype=dt)      # chunked host pipeline
            assert np.array_equal(d.cpu().numpy(), h), (kind, n_hash, dt)
        pi = torch.arange(0, 1000, 2, device=dev)
        estimate_pairs(d, pi, pi + 1)
        jaccard_block(d[:100], d[100:300])
        bucket_histogram(ids[:5000], fam, 4096)
# per-set and small-batch paths: the doorbell block (light requests), the launched
# (hash slice, set) grid with mapped or device staging, pinned and pageable outputs
from paper_1401_6124_b200 import FeatureSet, signature  # noqa: E402
from paper_1401_6124_b200.minhash import _signatures_csr_host  # noqa: E402

rng = np.random.default_rng(3)
for kind in ("iterative", "random"):
    for n_hash in (1, 128, 3000, 20_000):
        fam = make_family(kind, 9, n_hash, 1_048_583)
        for n in (1, 40, 900):
            s = FeatureSet(rng.integers(0, 1_048_583, size=n))
            signature(s, fam)
        for pinned in (False, True):
            buf = torch.empty((3, n_hash), dtype=torch.int64, pin_memory=pinned)
            _signatures_csr_host(np.array([0, 5, 5 + 700, 5 + 700 + 1], dtype=np.int64),
                                 rng.integers(0, 1_048_583, size=706).astype(np.uint32), fam, "int64", buf.numpy(),
                                 None)
torch.cuda.synchronize()
print("sanitize cases ok")
