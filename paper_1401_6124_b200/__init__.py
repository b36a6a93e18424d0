"""paper_1401_6124_b200 -- B200-native MinHash signatures (arXiv 1401.6124).

A drop-in for the reference package's signature path (``minhashlab``):
families, ``signature`` / ``estimate_jaccard`` and the signature files keep the
reference's API, while the per-set numba loops are replaced by sm_100a CUDA
kernels over CSR batches (``signatures_csr``) behind the C ABI in
``include/mhb.h`` (``lib/libmhb.so``).
"""
from .families import (
    FAMILY_KINDS,
    HashParams,
    IterativeFamily,
    RandomFamily,
    derive_seed,
    family_from_json,
    family_to_json,
    make_family,
    make_iterative_family,
    sample_random_family,
)
from .minhash import (
    FeatureSet,
    Signature,
    band_keys,
    signatures_band_keys,
    estimate_jaccard,
    estimate_pairs,
    exact_jaccard,
    jaccard_block,
    read_signatures_binary,
    read_signatures_text,
    sign_csr_device,
    signature,
    signatures,
    signatures_csr,
    write_signatures_binary,
    write_signatures_text,
)
from .modmath import MAX_KERNEL_PRIME, MAX_VECTOR_PRIME, choose_prime, is_prime, mulmod, next_prime
from .stats import bucket_histogram

__version__ = "0.1.0"

__all__ = [
    "FAMILY_KINDS", "HashParams", "IterativeFamily", "RandomFamily", "derive_seed", "family_from_json",
    "family_to_json", "make_family", "make_iterative_family", "sample_random_family", "FeatureSet",
    "Signature", "band_keys", "signatures_band_keys", "estimate_jaccard", "estimate_pairs", "exact_jaccard", "jaccard_block",
    "read_signatures_binary", "read_signatures_text", "sign_csr_device", "signature", "signatures",
    "signatures_csr", "write_signatures_binary", "write_signatures_text", "MAX_KERNEL_PRIME",
    "MAX_VECTOR_PRIME", "choose_prime", "is_prime", "mulmod", "next_prime", "bucket_histogram",
]
