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
torch.cuda.synchronize()
print("sanitize cases ok")
