"""e2e (host numpy in -> host numpy out) time of cfg2 for the current MHB_HOST_CHUNKS."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import gen, make_family, signatures_csr  # noqa: E402

cfg = gen.CONFIGS["cfg2"]
ip, ids = gen.make_csr(cfg, device="cuda:0")
fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
pin_in = os.environ.get("E2E_PAGEABLE_IN") != "1"
ip_pin = torch.empty(ip.numel(), dtype=torch.int64, pin_memory=pin_in)
ids_pin = torch.empty(ids.numel(), dtype=torch.int32, pin_memory=pin_in)
DT = os.environ.get("E2E_DTYPE", "uint32")
out_pin = torch.empty((ip.numel() - 1, fam.size), dtype=torch.int32 if DT == "uint32" else torch.int64,
                      pin_memory=os.environ.get("E2E_PAGEABLE") != "1")
ip_pin.copy_(ip)
ids_pin.copy_(ids.view(torch.int32))
a, b = ip_pin.numpy(), ids_pin.numpy().view(np.uint32)
o = out_pin.numpy().view(np.uint32) if DT == "uint32" else out_pin.numpy()
for _ in range(2):
    signatures_csr(a, b, fam, out_dtype=DT, out=o)
t = []
for _ in range(5):
    t0 = time.perf_counter()
    signatures_csr(a, b, fam, out_dtype=DT, out=o)
    t.append(time.perf_counter() - t0)
print(DT, "in", "pinned" if pin_in else "pageable", "out", "pageable" if os.environ.get("E2E_PAGEABLE") == "1" else "pinned",
      "nt", os.environ.get("MHB_HOST_NT", "1"), os.environ.get("MHB_HOST_CHUNKS", "16"), "chunks:", round(statistics.mean(t) * 1e3, 2), "ms", round(min(t) * 1e3, 2))
