// records.cu -- signature-file records formatted on the GPU.
//
// The reference writes one record per object (minhash.py:140-206):
//   text   : f"{id} {N} " + " ".join(ids) + "\n"            (write_signatures_text)
//   binary : <QQ id, N> then N little-endian u64 ids        (write_signatures_binary)
// These kernels produce the same bytes from a device signature block, so large
// batches stream HBM -> host -> file without a per-entry Python loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"

namespace mhb {

template <typename T>
__global__ void binary_records_kernel(const T* __restrict__ sig, int64_t n_sets, int32_t n_hash,
                                      const int64_t* __restrict__ obj_ids, int64_t first_id,
                                      unsigned long long* __restrict__ out) {
    const int64_t words = (int64_t)n_hash + 2;
    const int64_t total = n_sets * words;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = w / words;
        const int64_t k = w - r * words;
        unsigned long long v;
        if (k == 0) v = (unsigned long long)(obj_ids ? obj_ids[r] : first_id + r);
        else if (k == 1) v = (unsigned long long)n_hash;
        else v = (unsigned long long)(long long)sig[r * n_hash + (k - 2)];
        out[w] = v;  // x86 / sm_100a are little-endian: the bytes are the reference's "<Q"
    }
}

__device__ __forceinline__ int ndigits_u64(unsigned long long v) {
    int d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

__device__ __forceinline__ int ndigits_i64(long long v) {
    return v < 0 ? 1 + ndigits_u64((unsigned long long)(-(v + 1)) + 1) : ndigits_u64((unsigned long long)v);
}

__device__ __forceinline__ void put_i64(char* dst, long long v, int nd) {
    unsigned long long u;
    if (v < 0) {
        *dst++ = '-';
        --nd;
        u = (unsigned long long)(-(v + 1)) + 1;
    } else {
        u = (unsigned long long)v;
    }
    for (int i = nd - 1; i >= 0; --i) {
        dst[i] = (char)('0' + (u % 10));
        u /= 10;
    }
}

// Warp per record: text length "id N x0 x1 ... xN-1\n".
template <typename T>
__global__ void text_lengths_kernel(const T* __restrict__ sig, int64_t n_sets, int32_t n_hash,
                                    const int64_t* __restrict__ obj_ids, int64_t first_id, int64_t* __restrict__ lens) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp0; r < n_sets; r += nwarps) {
        long long len = 0;
        for (int k = lane; k < n_hash; k += 32) len += ndigits_i64((long long)sig[r * n_hash + k]) + 1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
        if (lane == 0) {
            const long long id = obj_ids ? obj_ids[r] : first_id + r;
            // "id" + ' ' + "N" + ' ' + entries (each followed by ' ' or '\n')
            lens[r] = ndigits_i64(id) + 1 + ndigits_u64((unsigned long long)n_hash) + 1 + len;
        }
    }
}

// Warp per record; offsets[r] = byte offset of record r (exclusive scan of lens).
template <typename T>
__global__ void text_records_kernel(const T* __restrict__ sig, int64_t n_sets, int32_t n_hash,
                                    const int64_t* __restrict__ obj_ids, int64_t first_id,
                                    const int64_t* __restrict__ offsets, char* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp0; r < n_sets; r += nwarps) {
        char* line = out + offsets[r];
        const long long id = obj_ids ? obj_ids[r] : first_id + r;
        const int nid = ndigits_i64(id), nn = ndigits_u64((unsigned long long)n_hash);
        if (lane == 0) {
            put_i64(line, id, nid);
            line[nid] = ' ';
            put_i64(line + nid + 1, n_hash, nn);
            line[nid + 1 + nn] = ' ';
        }
        long long pos = nid + 1 + nn + 1;
        for (int k0 = 0; k0 < n_hash; k0 += 32) {
            const int k = k0 + lane;
            const long long v = k < n_hash ? (long long)sig[r * n_hash + k] : 0;
            const int w = k < n_hash ? ndigits_i64(v) + 1 : 0;
            int incl = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (k < n_hash) {
                char* dst = line + pos + incl - w;
                put_i64(dst, v, w - 1);
                dst[w - 1] = (k + 1 == n_hash) ? '\n' : ' ';
            }
            pos += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

static int grid_for(int64_t work, int threads_per_unit) {
    DeviceInfo dev;
    if (current_device_info(&dev)) return -1;
    int64_t blocks = (work * threads_per_unit + 255) / 256;
    if (blocks > (int64_t)dev.sms * 16) blocks = (int64_t)dev.sms * 16;
    return blocks < 1 ? 1 : (int)blocks;
}

}  // namespace mhb

using namespace mhb;

extern "C" int mhb_format_binary_records(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                                         const int64_t* obj_ids, int64_t first_id, unsigned long long* out,
                                         void* stream) {
    clear_error();
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "signature records need n_hash >= 1");
    if (n_sets <= 0) return MHB_OK;
    const int blocks = grid_for(n_sets * ((int64_t)n_hash + 2), 1);
    if (blocks < 0) return MHB_ERR_CUDA;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sig_dtype == MHB_OUT_I64)
        binary_records_kernel<long long><<<blocks, 256, 0, st>>>(static_cast<const long long*>(sig), n_sets, n_hash,
                                                                 obj_ids, first_id, out);
    else if (sig_dtype == MHB_OUT_U32)
        binary_records_kernel<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(sig), n_sets, n_hash,
                                                                obj_ids, first_id, out);
    else
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    return cuda_check(cudaGetLastError(), "binary_records launch");
}

extern "C" int mhb_text_record_lengths(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                                       const int64_t* obj_ids, int64_t first_id, int64_t* lens, void* stream) {
    clear_error();
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "signature records need n_hash >= 1");
    if (n_sets <= 0) return MHB_OK;
    const int blocks = grid_for(n_sets, 32);
    if (blocks < 0) return MHB_ERR_CUDA;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sig_dtype == MHB_OUT_I64)
        text_lengths_kernel<long long><<<blocks, 256, 0, st>>>(static_cast<const long long*>(sig), n_sets, n_hash,
                                                               obj_ids, first_id, lens);
    else if (sig_dtype == MHB_OUT_U32)
        text_lengths_kernel<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(sig), n_sets, n_hash,
                                                              obj_ids, first_id, lens);
    else
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    return cuda_check(cudaGetLastError(), "text_lengths launch");
}

extern "C" int mhb_format_text_records(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                                       const int64_t* obj_ids, int64_t first_id, const int64_t* offsets, char* out,
                                       void* stream) {
    clear_error();
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "signature records need n_hash >= 1");
    if (n_sets <= 0) return MHB_OK;
    const int blocks = grid_for(n_sets, 32);
    if (blocks < 0) return MHB_ERR_CUDA;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sig_dtype == MHB_OUT_I64)
        text_records_kernel<long long><<<blocks, 256, 0, st>>>(static_cast<const long long*>(sig), n_sets, n_hash,
                                                               obj_ids, first_id, offsets, out);
    else if (sig_dtype == MHB_OUT_U32)
        text_records_kernel<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(sig), n_sets, n_hash,
                                                              obj_ids, first_id, offsets, out);
    else
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    return cuda_check(cudaGetLastError(), "text_records launch");
}
