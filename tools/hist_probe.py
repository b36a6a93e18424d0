"""Time the bucket-histogram kernels on cfg3/cfg4-shaped inputs (the distinct ids of the
workload x N members into 4096 bins) -- for ncu captures and A/B runs.

  python tools/hist_probe.py [cfg3|cfg4] [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1401_6124_b200 import bucket_histogram, gen, make_family  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind = sys.argv[3] if len(sys.argv) > 3 else "iterative"
cfg = gen.CONFIGS[name]
dev = torch.device("cuda", 0)
n_x = {"cfg3": 4_194_304, "cfg4": 60_921_506}.get(name, 1 << 22)
g = torch.Generator(device=dev).manual_seed(1)
xs = torch.randperm(cfg.vocab, device=dev, generator=g)[:n_x].sort().values.to(torch.uint32)
fam = make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
h = bucket_histogram(xs, fam, 4096)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    bucket_histogram(xs, fam, 4096)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
ev = n_x * fam.size
sms = torch.cuda.get_device_properties(dev).multi_processor_count
print(f"{name} {kind}: {n_x} x {fam.size} = {ev:.3e} evals in {ms:.3f} ms: {ev / ms / 1e9:.3f} Tevals/s, "
      f"{ev / (ms * 1e-3) / sms / 1.965e9:.2f} evals/clk/SM at 1965 MHz; total {int(h.sum())}")
