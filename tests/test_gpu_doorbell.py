"""GPU: the per-set / small-batch paths of the host entry (csrc/small.cu): the doorbell
server (doorbell_kernel) and the launched (hash slice, set) grid (sign_small_kernel).

signature(FeatureSet, family) -- the reference's per-set call (minhash.py:91-110) --
is served by one resident block that polls a request word in mapped host memory.
These tests cover its protocol rather than the arithmetic (the small-batch parity
tests in test_gpu_parity.py run through it too): relaunch after the idle exit,
concurrent callers, interleaving with the chunked pipeline and device-wide syncs,
release while running, and equality with the launched small kernel
(MHB_DOORBELL=0) in a fresh process; then the wide per-set calls of the reference's C6
loop (100,000 hashes) and the output targets (caller's pinned buffer written directly,
or the mapped stage copied).  Bar: bit-exact against the oracle.
"""
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import FeatureSet, make_family, signature, signatures_csr

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _sets(seed, n, lo=1, hi=300, p=1_048_583):
    rng = np.random.default_rng(seed)
    return [FeatureSet(rng.integers(0, p, size=int(rng.integers(lo, hi)))) for _ in range(n)]


def _want(sets, fam):
    ip = np.zeros(len(sets) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([len(s) for s in sets])
    ids = np.concatenate([s.ids for s in sets]).astype(np.uint32)
    return oracle.sign_family_csr(ip, ids, fam)


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_per_set_calls_and_relaunch_after_idle(cuda_device, kind):
    fam = make_family(kind, 11, 128, 1_048_583)
    sets = _sets(1, 60)
    want = _want(sets, fam)
    for k, s in enumerate(sets):
        if k % 15 == 14:
            time.sleep(0.005)  # > the 1 ms idle exit: the next call relaunches the server
        assert np.array_equal(signature(s, fam).mins, want[k]), k


def test_concurrent_callers(cuda_device):
    import torch

    fam = make_family("iterative", 5, 200, 16_777_259)
    sets = _sets(2, 200, p=16_777_259)
    want = _want(sets, fam)
    got = [None] * len(sets)
    errors = []

    def work(t):
        try:
            torch.cuda.set_device(cuda_device)
            for k in range(t, len(sets), 4):
                got[k] = signature(sets[k], fam).mins
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errors.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for k in range(len(sets)):
        assert np.array_equal(got[k], want[k]), k


def test_interleaved_with_batches_and_device_syncs(cuda_device):
    import torch

    from paper_1401_6124_b200 import gen

    fam = make_family("iterative", 9, 128, 1_048_583)
    indptr, ids = gen.cfg1_numpy(n_sets=3000, seed=4)
    want_batch = oracle.sign_family_csr(indptr, ids, fam)
    sets = _sets(3, 20)
    want = _want(sets, fam)
    for k, s in enumerate(sets):
        assert np.array_equal(signature(s, fam).mins, want[k])
        if k % 5 == 0:
            t0 = time.perf_counter()
            torch.cuda.synchronize()  # waits for the server's idle exit (<= 1 ms + slack)
            assert time.perf_counter() - t0 < 1.0
        if k % 7 == 0:
            got = signatures_csr(indptr, ids, fam, out_dtype="int64")  # chunked host pipeline
            assert np.array_equal(got, want_batch)


def test_release_while_running(cuda_device):
    from paper_1401_6124_b200 import _lib

    fam = make_family("random", 2, 64, 1_048_583)
    sets = _sets(4, 6)
    want = _want(sets, fam)
    for k, s in enumerate(sets):
        assert np.array_equal(signature(s, fam).mins, want[k])
        _lib.load().mhb_host_release()  # stops the resident block; the next call starts over


_CHILD = r"""
import numpy as np
from paper_1401_6124_b200 import FeatureSet, make_family, signature
rng = np.random.default_rng(8)
out = []
for kind, p in (("iterative", 1_048_583), ("random", 16_777_259), ("iterative", 4_294_967_291)):
    fam = make_family(kind, 3, 96, p)
    for _ in range(40):
        s = FeatureSet(rng.integers(0, p, size=int(rng.integers(1, 500))))
        out.append(signature(s, fam).mins)
np.save(__import__("sys").argv[1], np.concatenate(out))
"""


def test_doorbell_equals_launched_kernel(cuda_device, tmp_path):
    res = {}
    for mode in ("0", "1"):
        env = dict(os.environ, MHB_DOORBELL=mode, MHB_DOORBELL_IDLE_US="50",
                   PYTHONPATH=str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", ""))
        f = tmp_path / f"m{mode}.npy"
        subprocess.run([sys.executable, "-c", _CHILD, str(f)], check=True, env=env, cwd=ROOT, timeout=300)
        res[mode] = np.load(f)
    assert np.array_equal(res["0"], res["1"])


@pytest.mark.parametrize("kind", ["iterative", "random"])
def test_wide_per_set_calls(cuda_device, kind):
    """The reference's C6 call shape (one set, 100,000 hashes per signature() call): the
    launched (hash slice, set) grid, its result copied once into a fresh array."""
    p = 200_003
    fam = make_family(kind, 6, 100_000, p)
    sets = _sets(7, 6, lo=1, hi=400, p=p)
    want = _want(sets, fam)
    for k, s in enumerate(sets):
        got = signature(s, fam)
        assert got.mins.dtype == np.int64 and not got.mins.flags.writeable
        assert np.array_equal(got.mins, want[k]), k


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("n_hash", [300, 5000, 40_000])
def test_small_batch_output_targets(cuda_device, pinned, n_hash):
    """Small batches whose output is written into the caller's page-locked buffer directly,
    or into the mapped stage and copied (in parallel above 1 MB), both dtypes."""
    import torch

    from paper_1401_6124_b200.minhash import _signatures_csr_host

    fam = make_family("iterative", 8, n_hash, 1_048_583)
    sets = _sets(9, 40, p=1_048_583)
    want = _want(sets, fam)
    ip = np.zeros(len(sets) + 1, dtype=np.int64)
    ip[1:] = np.cumsum([len(s) for s in sets])
    ids = np.concatenate([s.ids for s in sets]).astype(np.uint32)
    for dt, tdt in (("int64", torch.int64), ("uint32", torch.int32)):
        buf = torch.empty((len(sets), n_hash), dtype=tdt, pin_memory=pinned)
        out = buf.numpy() if dt == "int64" else buf.numpy().view(np.uint32)
        got = _signatures_csr_host(ip, ids, fam, dt, out, None)
        assert got is out or np.shares_memory(got, out)
        assert np.array_equal(out.astype(np.int64), want), (dt, pinned, n_hash)


def test_wide_results_pinned_cap(cuda_device):
    """Retained wide per-set results stop being page-locked past MHB_PERSET_PINNED_MB, and
    dropped ones give their budget back."""
    import gc

    from paper_1401_6124_b200 import minhash

    fam = make_family("iterative", 2, 20_000, 1_048_583)
    s = _sets(12, 1, lo=30, hi=31)[0]
    want = _want([s], fam)[0]
    cap = minhash._PERSET_PINNED_CAP
    gc.collect()
    live0 = minhash._perset_pinned["live"]
    try:
        minhash._PERSET_PINNED_CAP = live0 + 3 * 8 * 20_000  # room for three more
        keep = [signature(s, fam) for _ in range(5)]
        assert all(np.array_equal(k.mins, want) for k in keep)
        assert minhash._perset_pinned["live"] == live0 + 3 * 8 * 20_000
        del keep
        gc.collect()
        assert minhash._perset_pinned["live"] == live0
    finally:
        minhash._PERSET_PINNED_CAP = cap
