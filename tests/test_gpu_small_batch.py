"""Small batches (<= 16,384 sets): the one-launch plan and sign_small_batch_kernel under
every lane count K and part count Q (MHB_SIGN_K / MHB_SMALL_Q are read once per process,
so each combination runs in its own interpreter: tests/_small_batch_check.py)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("K,Q", [(0, 0), (8, 1), (16, 2), (32, 4), (64, 1), (64, 4), (32, 1)])
def test_small_batch_kernel_lanes_and_parts(cuda_device, K, Q):
    env = dict(os.environ)
    if K:
        env["MHB_SIGN_K"] = str(K)
    if Q:
        env["MHB_SMALL_Q"] = str(Q)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "_small_batch_check.py"), str(K * 10 + Q)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout[-2000:] + r.stderr[-2000:]
