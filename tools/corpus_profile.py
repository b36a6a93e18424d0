"""Stage timings of the corpus ingest (GPU and host backends) on one synthetic corpus."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import derive_seed, gen  # noqa: E402
from paper_1401_6124_b200.corpus import build_corpus_csr  # noqa: E402

text = gen.synth_text_corpus(400000, derive_seed(gen.MASTER_SEED, 40), unicode_frac=float(sys.argv[1]) if len(sys.argv) > 1 else 0.01)
path = "/dev/shm/cp.txt"
open(path, "wb").write(text)
torch.cuda.init()
for backend in ("gpu", "host", "gpu"):
    t0 = time.perf_counter()
    build_corpus_csr(path, backend=backend)
    print(backend, round((time.perf_counter() - t0) * 1e3, 1), "ms")
t0 = time.perf_counter()
p = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
print("pinned alloc", round((time.perf_counter() - t0) * 1e3, 1), "ms")
cProfile.run("build_corpus_csr(path, backend='gpu')", "/tmp/cp.prof")
pstats.Stats("/tmp/cp.prof").sort_stats("tottime").print_stats(12)
