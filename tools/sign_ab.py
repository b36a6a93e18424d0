"""Time the signing kernel from several variant libraries in one process (a BASELINE
shape), interleaved over rounds: python tools/sign_ab.py cfg4 rounds lib1.so lib2.so ...
(MHB_AB_FAMILY=random: mhb_sign_random_csr)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import gen, make_family  # noqa: E402

name, rounds, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
cfg = gen.CONFIGS[name]
dev = torch.device("cuda", 0)
if name == "cfg3":
    ip, ids, _ = gen.planted_pairs(cfg, device=dev)
else:
    ip, ids = gen.make_csr(cfg, device=dev)
kind = os.environ.get("MHB_AB_FAMILY", "iterative")
fam = make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
if kind == "random":
    da, db = fam.device_params(dev)
n_sets, N = ip.numel() - 1, fam.size
out = torch.empty((n_sets, N), dtype=torch.uint32, device=dev)
P, I64, U64, I32, SZ = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_size_t
handles = []
for path in libs:
    lib = C.CDLL(path)
    lib.mhb_sign_workspace_bytes.restype = SZ
    lib.mhb_sign_workspace_bytes.argtypes = [I64, I64, I32]
    lib.mhb_sign_iterative_csr.restype = C.c_int
    lib.mhb_sign_iterative_csr.argtypes = [P, P, I64, I64, U64, U64, U64, I32, P, I32, P, P, SZ, P]
    lib.mhb_sign_random_csr.restype = C.c_int
    lib.mhb_sign_random_csr.argtypes = [P, P, I64, I64, P, P, U64, I32, P, I32, P, P, SZ, P]
    handles.append((path.split("/")[-1], lib))
ws_bytes = handles[0][1].mhb_sign_workspace_bytes(n_sets, ids.numel(), N)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
ref = None
res = {n: [] for n, _ in handles}
for r in range(rounds):
    for n, lib in handles:
        def call():
            if kind == "random":
                assert lib.mhb_sign_random_csr(ip.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), da.data_ptr(),
                                               db.data_ptr(), fam.prime, N, out.data_ptr(), 0, None, ws.data_ptr(),
                                               ws_bytes, st) == 0
                return
            assert lib.mhb_sign_iterative_csr(ip.data_ptr(), ids.data_ptr(), n_sets, ids.numel(), fam.base.a,
                                              fam.base.b, fam.prime, N, out.data_ptr(), 0, None, ws.data_ptr(),
                                              ws_bytes, st) == 0
        call()
        torch.cuda.synchronize()
        if r == 0:
            h = torch.sum(out.view(torch.int32).to(torch.int64)).item()
            ref = h if ref is None else ref
            assert h == ref, f"{n}: different signatures"
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            call()
        e1.record()
        torch.cuda.synchronize()
        res[n].append(e0.elapsed_time(e1) / 5)
for n, v in sorted(res.items(), key=lambda kv: min(kv[1])):
    print(f"{n:28s} " + " ".join(f"{x:.3f}" for x in v))
