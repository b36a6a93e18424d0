"""Bucket-uniformity histogram on the GPU.

The reference's uniformity experiment hashes one x through every family member
and counts buckets: ``np.bincount(family.eval_all(x) % buckets)`` (reference
stats.py:206-225).  ``bucket_histogram`` computes the same integer counts for a
whole batch of x values with the libmhb histogram kernel (exact: integer
counting, no sampling).  The chi-square / t-test math that consumes the counts
is microseconds of CPU work and stays out of scope.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .families import Family, IterativeFamily
from .modmath import MAX_KERNEL_PRIME


def bucket_histogram(xs, family: Family, buckets: int, counts=None):
    """counts[m] = #{(x, i): x in xs, i < N, h_i(x) mod buckets == m}, int64 on device.

    xs: CUDA tensor (or array-like, uploaded to the current device) of ids < prime.
    ``counts`` (int64 CUDA tensor of length ``buckets``) accumulates if given.  Any
    prime the reference accepts: primes >= 2^31 run the 64-bit-residue kernel."""
    import torch

    if buckets < 1:
        raise ValueError(f"need at least one bucket, got {buckets}")
    wide = family.prime > MAX_KERNEL_PRIME
    if not isinstance(xs, torch.Tensor) or not xs.is_cuda:
        arr = np.asarray(xs, dtype=np.int64).reshape(-1)
        if arr.size and (arr.min() < 0 or arr.max() >= family.prime):
            raise ValueError(f"hash input outside [0, {family.prime})")
        xs = torch.from_numpy(arr.astype(np.uint64 if wide else np.uint32)).cuda()
    # device tensors: ids < prime is the caller's precondition (no sync here)
    xs = xs.to(torch.int64).to(torch.uint64) if wide and xs.dtype != torch.uint64 else xs
    xs = (xs if wide else xs.to(torch.uint32)).contiguous()
    dev = xs.device
    if counts is None:
        counts = torch.zeros(buckets, dtype=torch.int64, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        if wide:
            if isinstance(family, IterativeFamily):
                rc = lib.mhb_bucket_hist_u64(_lib.KIND_ITERATIVE, xs.data_ptr(), xs.numel(), family.base.a,
                                             family.base.b, None, None, family.prime, family.size, buckets,
                                             counts.data_ptr(), stream)
            else:
                a, b = family.device_params(dev, wide=True)
                rc = lib.mhb_bucket_hist_u64(_lib.KIND_RANDOM, xs.data_ptr(), xs.numel(), 0, 0, a.data_ptr(),
                                             b.data_ptr(), family.prime, family.size, buckets, counts.data_ptr(),
                                             stream)
        elif isinstance(family, IterativeFamily):
            rc = lib.mhb_bucket_hist_iterative(xs.data_ptr(), xs.numel(), family.base.a, family.base.b,
                                               family.prime, family.size, buckets, counts.data_ptr(), stream)
        else:
            a, b = family.device_params(dev)
            rc = lib.mhb_bucket_hist_random(xs.data_ptr(), xs.numel(), a.data_ptr(), b.data_ptr(),
                                            family.prime, family.size, buckets, counts.data_ptr(), stream)
    _lib.check(rc)
    return counts
