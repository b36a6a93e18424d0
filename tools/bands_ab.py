"""A/B of the fused band-key epilogue: times sign only / fused / fused keys-only with
preallocated outputs (cfg4 shape), for the libmhb given by MHB_LIB (default in-tree)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import _lib, gen, make_family  # noqa: E402

n_sets = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
cfg = gen.CONFIGS["cfg4"]
dev = torch.device("cuda", 0)
ip, ids = gen.make_csr(cfg, device=dev, n_sets=n_sets)
fam = make_family("iterative", cfg.family_seed("iterative"), cfg.n_hash, cfg.prime)
lib = _lib.load()
N, rows = fam.size, 16
out = torch.empty((n_sets, N), dtype=torch.uint32, device=dev)
keys = torch.empty((n_sets, N // rows), dtype=torch.uint64, device=dev)
ws_bytes = lib.mhb_sign_workspace_bytes(n_sets, ids.numel(), N)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream


def sign():
    _lib.check(lib.mhb_sign_iterative_csr(ip.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), fam.base.a, fam.base.b,
                                          fam.prime, N, out.data_ptr(), 0, None, ws.data_ptr(), ws_bytes, st))


def fused(write):
    _lib.check(lib.mhb_sign_iterative_csr_bands(ip.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), fam.base.a,
                                                fam.base.b, fam.prime, N, rows, keys.data_ptr(), out.data_ptr(), 0,
                                                write, None, ws.data_ptr(), ws_bytes, st))


def t(fn, reps=8):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tag = os.environ.get("MHB_LIB", "in-tree").split("/")[-1]
print(f"{tag:12s} sign {t(sign):.3f} ms  fused {t(lambda: fused(1)):.3f} ms  keys-only {t(lambda: fused(0)):.3f} ms",
      flush=True)
