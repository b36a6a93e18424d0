"""Reference-facing API semantics that need no GPU (CPU only): FeatureSet,
Signature, estimate_jaccard / exact_jaccard, signature files, and the rule that
the signing path never falls back to the CPU."""
import struct

import numpy as np
import pytest

from paper_1401_6124_b200 import (
    FeatureSet,
    Signature,
    estimate_jaccard,
    exact_jaccard,
    make_family,
    read_signatures_binary,
    read_signatures_text,
    signatures_csr,
    write_signatures_binary,
    write_signatures_text,
)


def test_featureset_canonical():
    fs = FeatureSet([5, 1, 3, 1, 5])
    assert fs.ids.tolist() == [1, 3, 5] and len(fs) == 3 and list(fs) == [1, 3, 5]
    assert FeatureSet([3, 1, 2]) == FeatureSet([2, 3, 1, 1])
    assert len(FeatureSet([])) == 0
    with pytest.raises(ValueError):
        FeatureSet([1, -2])
    with pytest.raises(ValueError):
        FeatureSet([]).max_id


def test_signature_is_readonly_int64():
    sig = Signature(np.array([1, 2, 3], dtype=np.uint32), ("iterative", 1, 3, 7))
    assert sig.mins.dtype == np.int64 and not sig.mins.flags.writeable and len(sig) == 3


def test_estimate_jaccard_semantics():
    key = ("random", 1, 4, 7757)
    a = Signature(np.array([1, 2, 3, 4]), key)
    b = Signature(np.array([1, 2, 9, 9]), key)
    assert estimate_jaccard(a, b) == 0.5 and estimate_jaccard(a, a) == 1.0
    with pytest.raises(ValueError):
        estimate_jaccard(a, Signature(np.array([1, 2, 3, 4]), ("random", 2, 4, 7757)))
    with pytest.raises(ValueError):
        estimate_jaccard(a, Signature(np.array([1, 2, 3]), key))


def test_exact_jaccard():
    assert exact_jaccard(FeatureSet([]), FeatureSet([])) == 1.0
    assert exact_jaccard(FeatureSet([1, 2, 3]), FeatureSet([2, 3, 4])) == 0.5


def test_signature_files_round_trip(tmp_path):
    records = [(7, Signature(np.array([1, 2]))), (9, np.array([5, 6, 7]))]
    write_signatures_text(tmp_path / "s.txt", records)
    assert (tmp_path / "s.txt").read_text() == "7 2 1 2\n9 3 5 6 7\n"
    back = read_signatures_text(tmp_path / "s.txt")
    assert [(i, m.tolist()) for i, m in back] == [(7, [1, 2]), (9, [5, 6, 7])]
    write_signatures_binary(tmp_path / "s.bin", records[:1])
    assert (tmp_path / "s.bin").read_bytes() == struct.pack("<QQQQ", 7, 2, 1, 2)  # test_minhash.py:242-246
    assert [(i, m.tolist()) for i, m in read_signatures_binary(tmp_path / "s.bin")] == [(7, [1, 2])]


def test_truncated_files_rejected(tmp_path):
    (tmp_path / "t.txt").write_text("1 3 4 5\n")
    with pytest.raises(ValueError):
        read_signatures_text(tmp_path / "t.txt")
    (tmp_path / "t.bin").write_bytes(struct.pack("<QQQ", 1, 2, 3))
    with pytest.raises(ValueError):
        read_signatures_binary(tmp_path / "t.bin")


def test_no_cpu_fallback_for_signing():
    """CPU tensors are rejected: the signing path is CUDA-only by design."""
    import torch

    fam = make_family("iterative", 1, 8, 7757)
    with pytest.raises(ValueError, match="CUDA"):
        signatures_csr(torch.tensor([0, 2]), torch.tensor([1, 2], dtype=torch.int64), fam)


def test_out_of_range_inputs_rejected_before_cuda():
    """Checked on the host before any device work (so this runs on CPU)."""
    fam = make_family("iterative", 1, 8, 2**61 - 1)  # a wide prime: supported on the device
    with pytest.raises(ValueError):
        signatures_csr(np.array([0, 1]), np.array([2**61], dtype=np.int64), fam)  # id >= p
    with pytest.raises(ValueError):
        signatures_csr(np.array([0, 1]), np.array([-1], dtype=np.int64), fam)
