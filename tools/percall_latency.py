"""Per-call latency of the reference-style per-set API (signature) vs the batched path."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import FeatureSet, gen, make_family, signature, signatures_csr  # noqa: E402

indptr, ids = gen.cfg1_numpy(n_sets=2000, seed=3)
fam = make_family("iterative", 1, 128, 1_048_583)
sets = [FeatureSet(ids[indptr[s]:indptr[s + 1]]) for s in range(2000)]
torch.cuda.init()
for s in sets[:50]:
    signature(s, fam)
t0 = time.perf_counter()
for s in sets:
    signature(s, fam)
dt = (time.perf_counter() - t0) / len(sets)
print(f"signature(): {dt * 1e6:.1f} us/call (N=128, ~50 ids)")
one = np.array([0, len(sets[0])], dtype=np.int64)
x = sets[0].ids.astype(np.uint32)
for _ in range(50):
    signatures_csr(one, x, fam)
t0 = time.perf_counter()
for _ in range(2000):
    signatures_csr(one, x, fam)
print(f"signatures_csr(numpy, S=1): {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us/call")
signatures_csr(indptr, ids, fam)  # warm: staging buffers grow once
t0 = time.perf_counter()
for _ in range(20):
    signatures_csr(indptr, ids, fam)
print(f"signatures_csr(numpy, S=2000): {(time.perf_counter() - t0) * 1e6 / 20 / 2000:.3f} us/set")

import ctypes as C  # noqa: E402

from paper_1401_6124_b200 import _lib  # noqa: E402

lib = _lib.load()
out = np.empty(128, dtype=np.int64)
st = C.c_int32(0)
args = (_lib.KIND_ITERATIVE, one.ctypes.data, x.ctypes.data, 1, x.size, fam.base.a, fam.base.b, None, None,
        fam.prime, 128, out.ctypes.data, _lib.OUT_I64, C.addressof(st), 0)
for _ in range(100):
    lib.mhb_sign_csr_host(*args)
t0 = time.perf_counter()
for _ in range(5000):
    lib.mhb_sign_csr_host(*args)
print(f"raw mhb_sign_csr_host (S=1): {(time.perf_counter() - t0) / 5000 * 1e6:.1f} us/call")
import cProfile, pstats  # noqa: E402,E401

cProfile.run("for s in sets[:500]: signature(s, fam)", "/tmp/sig.prof")  # noqa: E702
pstats.Stats("/tmp/sig.prof").sort_stats("tottime").print_stats(10)

# the reference's timing experiment calls signature() once per document with N = 100,000
# (run_timing, bench.py:97-102; acceptance C6): per-document latency at that width
from paper_1401_6124_b200 import derive_seed  # noqa: E402

c6_ip, c6_ids, c6_p, c6_seed = gen.c6_workload()
c6_sets = [FeatureSet(c6_ids[c6_ip[s]:c6_ip[s + 1]]) for s in range(c6_ip.size - 1)]
for kind in ("iterative", "random"):
    fam = make_family(kind, derive_seed(c6_seed, 0), 100_000, c6_p)
    for s in c6_sets[:20]:
        signature(s, fam)
    t0 = time.perf_counter()
    for s in c6_sets:
        signature(s, fam)
    dt = time.perf_counter() - t0
    print(f"C6 per-document signature() {kind}: {dt / len(c6_sets) * 1e6:.1f} us/doc, {dt * 1e3:.1f} ms for {len(c6_sets)} docs")
