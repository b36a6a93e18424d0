"""GPU: the signing launch sequence (plan kernels, sign_kernel, finalize) is capturable
as one CUDA graph and its replays equal eager signing (bench.py --graph replays it for
launch-bound batches).  Bar: bit-exact against the oracle."""
import numpy as np
import pytest

from oracle import oracle
from paper_1401_6124_b200 import gen, make_family
from paper_1401_6124_b200.minhash import sign_csr_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n_hash", [("iterative", 128), ("random", 128), ("iterative", 2048)])
def test_graph_replay_equals_oracle(cuda_device, kind, n_hash):
    import torch

    indptr, ids = gen.cfg1_numpy(n_sets=3000, seed=21)
    fam = make_family(kind, 4, n_hash, 1_048_583)
    want = oracle.sign_family_csr(indptr, ids, fam)
    ip = torch.as_tensor(indptr, device=cuda_device)
    di = torch.as_tensor(ids.astype(np.int64), device=cuda_device).to(torch.uint32)
    out = torch.zeros((indptr.size - 1, n_hash), dtype=torch.int32, device=cuda_device)
    status = torch.zeros(1, dtype=torch.int32, device=cuda_device)

    def step():
        sign_csr_device(ip, di, fam, out, status, torch.cuda.current_stream())

    side = torch.cuda.Stream(cuda_device)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        assert np.array_equal(out.cpu().numpy().view(np.uint32).astype(np.int64), want)
