// wide.cu -- signatures for primes 2^31 <= p < 2^63 (64-bit residues).
//
// The u32 kernels (sign.cu) cover every BASELINE prime.  The reference also signs
// with larger primes: its numba kernels run up to MAX_VECTOR_PRIME = 3,037,000,499
// and `_signature_by_rows` beyond (minhash.py:102-127).  This path keeps the
// drop-in complete for those: 128-bit products, 64-bit walk, argmin tracked
// directly with the reference's tie rule (smaller id wins on equal hashes,
// kernels.py:23-26), so no inverse is needed.  Correctness first: one thread per
// (set, block of kWideLanes hash lanes).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"
#include "sign_internal.h"

namespace mhb {

constexpr int kWideLanes = 8;

__device__ __forceinline__ uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t p) {
    return (uint64_t)(((unsigned __int128)a * b) % p);
}

__device__ __forceinline__ uint64_t addmod64(uint64_t a, uint64_t b, uint64_t p) {
    const uint64_t t = a + b;  // a, b < p < 2^63: no overflow
    return t >= p ? t - p : t;
}

template <bool ITER, typename OutT, typename IdT>
__global__ void sign_wide_kernel(const int64_t* __restrict__ indptr, const IdT* __restrict__ ids,
                                 int64_t n_sets, uint64_t a, uint64_t b, const uint64_t* __restrict__ ra,
                                 const uint64_t* __restrict__ rb, uint64_t p, int32_t n_hash, OutT* __restrict__ out,
                                 int32_t* status) {
    const int blocks_per_set = (n_hash + kWideLanes - 1) / kWideLanes;
    const int64_t units = n_sets * blocks_per_set;
    bool bad = false;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = u / blocks_per_set;
        const int i0 = (int)(u - s * blocks_per_set) * kWideLanes;
        const int nl = min(kWideLanes, n_hash - i0);
        const int64_t lo = indptr[s], hi = indptr[s + 1];
        if (hi <= lo) continue;
        uint64_t best[kWideLanes], arg[kWideLanes];
#pragma unroll
        for (int k = 0; k < kWideLanes; ++k) {
            best[k] = ~0ull;
            arg[k] = ~0ull;
        }
        for (int64_t j = lo; j < hi; ++j) {
            const uint64_t x = ids[j];
            bad |= x >= p;
            if (ITER) {
                // h_{i0}(x) = (a+i0) x + i0 b mod p, then h <- h + (x+b) mod p (families.py:124-176)
                const uint64_t dh = addmod64(x % p, b, p);
                uint64_t h = addmod64(mulmod64((a + (uint64_t)i0) % p, x, p), mulmod64((uint64_t)i0, b, p), p);
#pragma unroll
                for (int k = 0; k < kWideLanes; ++k) {
                    if (k < nl && (h < best[k] || (h == best[k] && x < arg[k]))) {
                        best[k] = h;
                        arg[k] = x;
                    }
                    h = addmod64(h, dh, p);
                }
            } else {
#pragma unroll
                for (int k = 0; k < kWideLanes; ++k) {
                    if (k < nl) {
                        const uint64_t h = addmod64(mulmod64(ra[i0 + k], x, p), rb[i0 + k], p);
                        if (h < best[k] || (h == best[k] && x < arg[k])) {
                            best[k] = h;
                            arg[k] = x;
                        }
                    }
                }
            }
        }
        OutT* row = out + s * (int64_t)n_hash + i0;
        for (int k = 0; k < nl; ++k) row[k] = (OutT)arg[k];
    }
    if (bad && status) atomicOr(status, MHB_STATUS_ID_GE_PRIME);
}

__global__ void wide_check_kernel(const int64_t* __restrict__ indptr, int64_t n_sets, const uint64_t* ra,
                                  const uint64_t* rb, int32_t n_hash, uint64_t p, int32_t* status) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = tid; s < n_sets; s += stride)
        if (indptr[s + 1] <= indptr[s] && status) atomicOr(status, MHB_STATUS_EMPTY_SET);
    if (ra)
        for (int64_t i = tid; i < n_hash; i += stride)
            if ((ra[i] == 0 || ra[i] >= p || rb[i] >= p) && status) atomicOr(status, MHB_STATUS_BAD_PARAM);
}

template <typename IdT>
int launch_sign_wide_t(bool iter, const int64_t* indptr, const IdT* ids, int64_t n_sets, uint64_t a, uint64_t b,
                       const uint64_t* ra, const uint64_t* rb, uint64_t prime, int32_t n_hash, void* out,
                       int32_t out_dtype, int32_t* status, cudaStream_t st) {
    if (status) {
        int rc = cuda_check(cudaMemsetAsync(status, 0, sizeof(int32_t), st), "memset status");
        if (rc) return rc;
    }
    if (n_sets == 0) return MHB_OK;
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    wide_check_kernel<<<dev.sms, 256, 0, st>>>(indptr, n_sets, iter ? nullptr : ra, rb, n_hash, prime, status);
    const int64_t units = n_sets * ((n_hash + kWideLanes - 1) / kWideLanes);
    int64_t blocks = (units + 127) / 128;
    if (blocks > (int64_t)dev.sms * 16) blocks = (int64_t)dev.sms * 16;
    if (blocks < 1) blocks = 1;
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (iter && i64)
        sign_wide_kernel<true, long long, IdT><<<(unsigned)blocks, 128, 0, st>>>(
            indptr, ids, n_sets, a, b, ra, rb, prime, n_hash, static_cast<long long*>(out), status);
    else if (iter)
        sign_wide_kernel<true, uint32_t, IdT><<<(unsigned)blocks, 128, 0, st>>>(
            indptr, ids, n_sets, a, b, ra, rb, prime, n_hash, static_cast<uint32_t*>(out), status);
    else if (i64)
        sign_wide_kernel<false, long long, IdT><<<(unsigned)blocks, 128, 0, st>>>(
            indptr, ids, n_sets, a, b, ra, rb, prime, n_hash, static_cast<long long*>(out), status);
    else
        sign_wide_kernel<false, uint32_t, IdT><<<(unsigned)blocks, 128, 0, st>>>(
            indptr, ids, n_sets, a, b, ra, rb, prime, n_hash, static_cast<uint32_t*>(out), status);
    return cuda_check(cudaGetLastError(), "sign_wide launch");
}

int launch_sign_wide(bool iter, const int64_t* indptr, const uint32_t* ids, int64_t n_sets, uint64_t a, uint64_t b,
                     const uint64_t* ra, const uint64_t* rb, uint64_t prime, int32_t n_hash, void* out,
                     int32_t out_dtype, int32_t* status, cudaStream_t st) {
    return launch_sign_wide_t<uint32_t>(iter, indptr, ids, n_sets, a, b, ra, rb, prime, n_hash, out, out_dtype,
                                        status, st);
}

}  // namespace mhb

extern "C" int mhb_sign_random_csr_u64(const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t nnz,
                                       const uint64_t* a, const uint64_t* b, uint64_t prime, int32_t n_hash,
                                       void* out, int32_t out_dtype, int32_t* status, void* stream) {
    using namespace mhb;
    clear_error();
    if (n_sets < 0 || nnz < 0) return set_error(MHB_ERR_INVALID, "n_sets and nnz must be >= 0");
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function, got %d", n_hash);
    if (prime < 3 || !is_prime_u64(prime)) return set_error(MHB_ERR_INVALID, "modulus %llu is not prime",
                                                             (unsigned long long)prime);
    if (prime >= (1ull << 63)) return set_error(MHB_ERR_UNSUPPORTED, "prime >= 2^63 is out of range");
    if (out_dtype != MHB_OUT_U32 && out_dtype != MHB_OUT_I64)
        return set_error(MHB_ERR_INVALID, "unknown out_dtype %d", out_dtype);
    if (!a || !b) return set_error(MHB_ERR_INVALID, "random family needs device arrays a and b");
    return launch_sign_wide(false, indptr, ids, n_sets, 0, 0, a, b, prime, n_hash, out, out_dtype, status,
                            static_cast<cudaStream_t>(stream));
}

// 64-bit feature ids (the reference's int64 FeatureSet ids; with primes >= 2^32 they
// may exceed 2^32): any prime < 2^63, int64 output.
extern "C" int mhb_sign_csr_ids64(int32_t kind, const int64_t* indptr, const uint64_t* ids, int64_t n_sets,
                                  int64_t nnz, uint64_t a, uint64_t b, const uint64_t* ra, const uint64_t* rb,
                                  uint64_t prime, int32_t n_hash, long long* out, int32_t* status, void* stream) {
    using namespace mhb;
    clear_error();
    if (kind != KIND_ITERATIVE && kind != KIND_RANDOM) return set_error(MHB_ERR_INVALID, "unknown kind %d", kind);
    if (n_sets < 0 || nnz < 0) return set_error(MHB_ERR_INVALID, "n_sets and nnz must be >= 0");
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function, got %d", n_hash);
    if (prime < 3 || !is_prime_u64(prime)) return set_error(MHB_ERR_INVALID, "modulus %llu is not prime",
                                                             (unsigned long long)prime);
    if (prime >= (1ull << 63)) return set_error(MHB_ERR_UNSUPPORTED, "prime >= 2^63 is out of range");
    if (kind == KIND_ITERATIVE) {
        if (a < 1 || a >= prime || b >= prime) return set_error(MHB_ERR_INVALID, "need 1 <= a < p and 0 <= b < p");
        if (a + (uint64_t)n_hash >= prime)
            return set_error(MHB_ERR_INVALID, "need a + size < prime to keep every member invertible");
    } else if (!ra || !rb) {
        return set_error(MHB_ERR_INVALID, "random family needs device arrays a and b");
    }
    if (n_sets > 0 && (!indptr || !out)) return set_error(MHB_ERR_INVALID, "null indptr/out");
    if (nnz > 0 && !ids) return set_error(MHB_ERR_INVALID, "null ids");
    return launch_sign_wide_t<uint64_t>(kind == KIND_ITERATIVE, indptr, ids, n_sets, a, b, ra, rb, prime, n_hash,
                                        out, MHB_OUT_I64, status, static_cast<cudaStream_t>(stream));
}
