// host_internal.h -- shared by host.cu (the chunked host-buffer pipeline of
// mhb_sign_csr_host) and small.cu (its small-batch paths: the resident doorbell block
// and the launched (hash slice, set) grid).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace mhb {

// host-memory helpers (host.cu)
bool is_pinned(const void* p);                            // page-locked host memory
bool is_device_ptr(const void* p);                        // device (or managed) memory
int grow(void** ptr, size_t* cap, size_t need);           // device buffer, grown on demand
// parallel (parts of >= part_elems elements), streaming stores
void host_copy_out(const uint32_t* src, void* dst, int64_t n, bool widen, int64_t part_elems = 1 << 18);

// Small batches (the per-set reference API: signature() on one FeatureSet) skip the
// chunk pipeline.  Light requests go to the resident doorbell block (no launch): inputs
// and outputs stay in mapped pinned memory.  Heavier ones (the reference's C6 timing
// loop: one set, 100,000 hashes per call) take one launch of sign_small_kernel over
// (hash slice, set) blocks, through device memory with one DMA each way when the output
// is wide.  A page-locked caller buffer receives its result directly; otherwise a
// mapped stage is copied out on the host.
constexpr int64_t kSmallSets = 64;
constexpr int64_t kSmallNnz = 1 << 16;
constexpr int64_t kSmallSetMax = 8192;     // ids of one set in shared memory
constexpr int64_t kSmallEntries = 1 << 21;  // n_sets * n_hash (16 MB of int64 output)
constexpr int32_t kSmallSliceHashes = 256;  // hashes per block of sign_small_kernel
constexpr int64_t kSmallStatus = kSmallEntries / kSmallSliceHashes + kSmallSets;  // >= its blocks

struct Doorbell;  // small.cu

struct SmallStage {
    char* in = nullptr;    // indptr | ids | a | b   (mapped pinned, grown on demand)
    size_t in_cap = 0;
    char* out = nullptr;   // [sets, hashes] u32 / i64 (mapped pinned, grown on demand)
    size_t out_cap = 0;
    int32_t* status = nullptr;  // kSmallStatus words (mapped pinned): one per block of sign_small_kernel
    void* dev = nullptr;        // device stage of wide launched batches: request | output | status
    size_t dev_cap = 0;
    Doorbell* db = nullptr;          // mapped pinned control block of the doorbell server
    char* req = nullptr;             // mapped pinned packed request (kDoorbellBytes)
    cudaStream_t db_stream = nullptr;  // the server's own non-blocking stream
    uint32_t seq = 0;                // last request number posted (and served)
};

// small.cu
bool small_batch(const int64_t* indptr, int64_t n_sets, int32_t n_hash, uint64_t prime);
int sign_small(SmallStage& sm, cudaStream_t stream, int32_t kind, const int64_t* indptr, const uint32_t* ids,
               int64_t n_sets, uint64_t a, uint64_t b, const uint32_t* a_host, const uint32_t* b_host,
               bool params_dev, uint64_t prime, int32_t n_hash, void* out, int32_t out_dtype,
               int32_t* status_host);
void small_release(SmallStage& sm);  // stops the doorbell block, frees the stages

}  // namespace mhb
