"""cProfile of corpus.sign_corpus on a synthetic corpus (where the non-ingest time goes)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_6124_b200 import derive_seed, gen  # noqa: E402
from paper_1401_6124_b200.corpus import sign_corpus  # noqa: E402

text = gen.synth_text_corpus(400000, derive_seed(gen.MASTER_SEED, 40), unicode_frac=0.01)
open("/dev/shm/sc.txt", "wb").write(text)
for _ in range(2):
    sign_corpus("/dev/shm/sc.txt", "/dev/shm/sc.out", family="iterative", hashes=128, log=None)
torch.cuda.synchronize()
t0 = time.perf_counter()
sign_corpus("/dev/shm/sc.txt", "/dev/shm/sc.out", family="iterative", hashes=128, log=None)
print("sign_corpus", (time.perf_counter() - t0) * 1e3, "ms")
cProfile.run('sign_corpus("/dev/shm/sc.txt", "/dev/shm/sc.out", family="iterative", hashes=128, log=None)', "/tmp/sc.prof")
pstats.Stats("/tmp/sc.prof").sort_stats("tottime").print_stats(18)
