"""Per-call latency of the reference's own signature() (numba) at the cfg1 shape.

Build container only (the reference is not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/reference_percall.py
The same 2,000 sets as bench.py's per_set entry (gen.cfg1_numpy(2000, seed=3)).
"""
import sys, time, numpy as np
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from paper_1401_6124_b200 import gen
from minhashlab import minhash, families
ip, ids = gen.cfg1_numpy(n_sets=2000, seed=3)
cfg = gen.CONFIGS["cfg1"]
sets = [minhash.FeatureSet(ids[ip[k]:ip[k+1]].astype(np.int64)) for k in range(2000)]
for kind in ("iterative", "random"):
    fam = families.make_family(kind, cfg.family_seed(kind), cfg.n_hash, cfg.prime)
    for s in sets[:100]: minhash.signature(s, fam)
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        for s in sets: minhash.signature(s, fam)
        best = min(best, (time.perf_counter() - t0) / len(sets) * 1e6)
    print(f"reference minhashlab.signature() {kind}: {best:.1f} us/call (N={cfg.n_hash}, mean {np.diff(ip).mean():.1f} ids), this container's CPU")
