// host.cu -- host-buffer entry point: chunked, copy/compute-overlapped signing.
//
// The reference's callers hand numpy arrays to the signing loop and get numpy
// arrays back (minhash.py:91-110, bench.py:97-102).  mhb_sign_csr_host is the
// native equivalent for a whole CSR batch living in host memory: the sets are
// cut into nnz-balanced chunks; each chunk goes H2D -> sign kernels -> D2H on
// one of kLanes streams, so the copy engines (both directions) and the SMs
// work on different chunks at the same time.  Device buffers are cached per
// device between calls (mhb_host_release frees them).
#include <cuda_runtime.h>

#include <algorithm>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <chrono>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

namespace {

constexpr int kLanes = 4;
constexpr int kMaxChunks = 4096;

struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;  // recorded after the lane's last D2H
    int64_t* indptr = nullptr;
    size_t indptr_cap = 0;
    uint32_t* ids = nullptr;
    size_t ids_cap = 0;
    void* out = nullptr;
    size_t out_cap = 0;
    void* ws = nullptr;
    size_t ws_cap = 0;
    // pinned staging for pageable caller buffers / int64 output (see mhb_sign_csr_host)
    uint32_t* stage_ids = nullptr;
    size_t stage_ids_cap = 0;
    uint32_t* stage_out = nullptr;
    size_t stage_out_cap = 0;
    int64_t pend_s0 = -1, pend_rows = 0;  // chunk whose staged output awaits the host copy
};

// Persistent host worker pool for the staging copies (page-cache-speed memcpy and the
// u32 -> int64 widening run on many cores while the GPU moves the next chunks).
class HostPool {
  public:
    HostPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int n = (int)std::min(16u, hw) - 1;  // the calling thread works too
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // fn(part) for part in [0, parts), spread over the pool and the caller
    void run(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1 || th_.empty()) {
            for (int k = 0; k < parts; ++k) fn(k);
            return;
        }
        {
            std::lock_guard<std::mutex> l(m_);
            fn_ = &fn;
            parts_ = parts;
            next_.store(0);
            left_ = parts;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [this] { return left_ == 0; });
        fn_ = nullptr;
    }
    int width() const { return (int)th_.size() + 1; }

  private:
    void work() {
        for (int k; (k = next_.fetch_add(1)) < parts_;) {
            (*fn_)(k);
            std::lock_guard<std::mutex> l(m_);
            if (--left_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int parts_ = 0, left_ = 0;
    std::atomic<int> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

HostPool& host_pool() {
    static HostPool pool;
    return pool;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int grow_pinned(void** ptr, size_t* cap, size_t need) {
    if (*cap >= need && *ptr) return MHB_OK;
    if (*ptr) cudaFreeHost(*ptr);
    *ptr = nullptr;
    *cap = 0;
    const size_t want = need + need / 4 + 256;
    int rc = cuda_check(cudaHostAlloc(ptr, want, cudaHostAllocDefault), "cudaHostAlloc (staging)");
    if (rc) return rc;
    *cap = want;
    return MHB_OK;
}

// Non-temporal (streaming) stores for the staging copies: the destination is written
// once and not read back by this CPU (a DMA source, or the caller's result), so the
// stores skip the read-for-ownership of every destination line.  SSE2 is baseline
// x86-64.  MHB_HOST_NT=0 uses plain stores (A/B: tools/e2e_chunks.py).
bool host_nt() {
    static const bool on = [] {
        const char* e = std::getenv("MHB_HOST_NT");
        return !(e && e[0] == '0');
    }();
    return on;
}

// dst[i] = src[i] (widen: as int64) for i in [0, n), streaming stores once dst is 16-byte aligned.
void copy_span(const uint32_t* src, void* dst_v, int64_t n, bool widen, bool nt) {
    int64_t i = 0;
#if defined(__SSE2__)
    if (nt) {
        if (widen) {
            long long* d = static_cast<long long*>(dst_v);
            for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = (long long)src[i];
            const __m128i z = _mm_setzero_si128();
            for (; i + 4 <= n; i += 4) {
                const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), _mm_unpacklo_epi32(v, z));
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 2), _mm_unpackhi_epi32(v, z));
            }
            for (; i < n; ++i) d[i] = (long long)src[i];
        } else {
            uint32_t* d = static_cast<uint32_t*>(dst_v);
            for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = src[i];
            for (; i + 8 <= n; i += 8) {
                const __m128i v0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
                const __m128i v1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 4));
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), v0);
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4), v1);
            }
            for (; i < n; ++i) d[i] = src[i];
        }
        _mm_sfence();  // order the streaming stores before the pool's completion signal
        return;
    }
#endif
    if (widen) {
        long long* d = static_cast<long long*>(dst_v);
        for (; i < n; ++i) d[i] = (long long)src[i];
    } else {
        std::memcpy(dst_v, src, (size_t)n * 4);
    }
}

bool direct_i64() {
    static const bool on = [] {
        const char* e = std::getenv("MHB_DIRECT_I64");
        return e && e[0] == '1';
    }();
    return on;
}

// Parallel copy (u32 -> u32, or u32 -> int64 widening) of `n` elements.
void host_copy_out(const uint32_t* src, void* dst, int64_t n, bool widen) {
    HostPool& pool = host_pool();
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool.width() * 2, n >> 18));
    const bool nt = host_nt();
    pool.run(parts, [&](int k) {
        const int64_t lo = n * k / parts, hi = n * (k + 1) / parts;
        char* d = static_cast<char*>(dst) + (size_t)lo * (widen ? 8 : 4);
        copy_span(src + lo, d, hi - lo, widen, nt);
    });
}

void host_copy_in(const uint32_t* src, uint32_t* dst, int64_t n) {
    HostPool& pool = host_pool();
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool.width() * 2, n >> 18));
    const bool nt = host_nt();
    pool.run(parts, [&](int k) {
        const int64_t lo = n * k / parts, hi = n * (k + 1) / parts;
        copy_span(src + lo, dst + lo, hi - lo, false, nt);
    });
}

// Small batches (the per-set reference API: signature() on one FeatureSet) skip the
// chunk pipeline.  Inputs are staged in mapped pinned memory and read over PCIe (ids
// once into shared memory); every (set, hash) argmin is computed exactly and written
// straight into mapped memory: the caller's own buffer when it is page-locked, else a
// mapped stage copied out on the host.  Light requests go to the resident doorbell
// block (no launch); heavier ones (the reference's C6 timing loop: one set, 100,000
// hashes per call) to one launch of sign_small_kernel over (hash slice, set) blocks.
constexpr int64_t kSmallSets = 64;
constexpr int64_t kSmallNnz = 1 << 16;
constexpr int64_t kSmallSetMax = 8192;     // ids of one set in shared memory
constexpr int64_t kSmallEntries = 1 << 21;  // n_sets * n_hash (16 MB of int64 output)
constexpr int32_t kSmallSliceHashes = 256;  // hashes per block of sign_small_kernel
constexpr int64_t kSmallStatus = kSmallEntries / kSmallSliceHashes + kSmallSets;  // >= its blocks

struct Doorbell;

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

struct DeviceCache {
    bool init = false;
    SmallStage small;
    Lane lanes[kLanes];
    int32_t* status = nullptr;  // one word per chunk, read once at the end
    uint32_t* ra = nullptr;
    uint32_t* rb = nullptr;
    size_t ra_cap = 0;
    size_t rb_cap = 0;
};

std::mutex g_mu;
DeviceCache g_cache[64];

// indptr[i] -= base: a chunk's CSR offsets become relative to its own ids buffer.
__global__ void rebase_indptr_kernel(int64_t* indptr, int64_t n, int64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        indptr[i] -= base;
}

// v mod p for v < 2^53 and floor(v / p), exactly, without a 64-bit integer division:
// a double-precision quotient estimate (off by at most one) and an integer correction.
__device__ __forceinline__ uint64_t mod_small(uint64_t v, uint64_t p, double inv_p) {
    const uint64_t q = (uint64_t)((double)v * inv_p);
    int64_t r = (int64_t)(v - q * p);
    if (r < 0) r += (int64_t)p;
    if (r >= (int64_t)p) r -= (int64_t)p;
    return (uint64_t)r;
}
// floor(A * 2^32 / p) for A < p < 2^31 (the Shoup companion of A), exactly.
__device__ __forceinline__ uint32_t shoup_of(uint64_t A, uint64_t p, double inv_p) {
    uint64_t q = (uint64_t)(ldexp((double)A, 32) * inv_p);  // < 2^32, off by at most one
    int64_t r = (int64_t)((A << 32) - q * p);               // true value in (-2p, 2p)
    while (r < 0) { r += (int64_t)p; --q; }
    while (r >= (int64_t)p) { r -= (int64_t)p; ++q; }
    return (uint32_t)q;
}
// (A x + B) mod p for A, B < p < 2^32, x < 2^32: A x + B < 2^64, quotient estimated in
// double (relative error ~2^-51 on a quotient < 2^33: off by at most a few), corrected.
__device__ __forceinline__ uint64_t mul_add_mod64(uint64_t A, uint64_t B, uint32_t x, uint64_t p, double inv_p) {
    const uint64_t v = A * x + B;
    const uint64_t q = (uint64_t)((double)A * (double)x * inv_p);
    int64_t r = (int64_t)(v - q * p);  // true value within a few p of [0, p)
    while (r < 0) r += (int64_t)p;
    while (r >= (int64_t)p) r -= (int64_t)p;
    return (uint64_t)r;
}

// Every hash of one set whose ids are already in shared memory, computed by one block
// exactly (u32 Shoup lanes for p < 2^31, 64-bit residues up to 2^32).  S = threads per
// hash (a power of two <= 32, from the block size and n_hash): each walks every S-th id
// (four independent minima for ILP) and the S partial minima meet in a shuffle
// reduction of (h << 32 | x) -- h is unique per distinct x (bijection on [0, p)), so
// the smallest key is the reference's argmin.  ra/rb: the random family's parameters
// (any address space).  Returns this thread's status flags.
__device__ __forceinline__ int small_set_hashes(const uint32_t* xs, int n, int kind, uint64_t a, uint64_t b,
                                                const uint32_t* ra, const uint32_t* rb, uint64_t p, int32_t n_hash,
                                                int32_t i_begin, int32_t i_end, void* out, int32_t out_dtype,
                                                int64_t set) {
    const int T = blockDim.x;  // a multiple of 32
    int S = 1;
    while (S < 32 && 2 * S * (i_end - i_begin) <= T && 2 * S <= n) S *= 2;
    const int per_round = T / S, slice = threadIdx.x % S;
    const double inv_p = 1.0 / (double)p;
    int flags = 0;
    for (int i0 = i_begin; i0 < i_end; i0 += per_round) {  // uniform trip count: whole warps shuffle below
        const int i = i0 + threadIdx.x / S;
        unsigned long long key = ~0ull;
        if (i < i_end) {
            uint64_t A, B;
            if (kind == KIND_ITERATIVE) {  // h_i(x) = ((a + i) x + i b) mod p, families.py:170-176
                A = a + (uint64_t)i;
                B = mod_small((uint64_t)i * b, p, inv_p);  // i < 2^14, b < 2^32
            } else {  // h_i(x) = (a_i x + b_i) mod p, kernels.py:21-41
                A = ra[i];
                B = rb[i];
                if (slice == 0 && (A < 1 || A >= p || B >= p)) flags |= MHB_STATUS_BAD_PARAM;
            }
            unsigned long long k1 = ~0ull, k2 = ~0ull, k3 = ~0ull;
            if (p < (1ull << 31)) {  // u32 Shoup multiply (modarith.cuh), exact for any x < 2^32
                const uint32_t a32 = (uint32_t)A, b32 = (uint32_t)B, p32 = (uint32_t)p;
                const uint32_t ap = shoup_of(A, p, inv_p);
                auto h = [&](uint32_t x) {
                    return ((unsigned long long)mul_add_mod(a32, ap, b32, x, p32) << 32) | x;
                };
                int k = slice;
                for (; k + 3 * S < n; k += 4 * S) {
                    const unsigned long long h0 = h(xs[k]), h1 = h(xs[k + S]), h2 = h(xs[k + 2 * S]),
                                             h3 = h(xs[k + 3 * S]);
                    key = h0 < key ? h0 : key;
                    k1 = h1 < k1 ? h1 : k1;
                    k2 = h2 < k2 ? h2 : k2;
                    k3 = h3 < k3 ? h3 : k3;
                }
                for (; k < n; k += S) {
                    const unsigned long long h0 = h(xs[k]);
                    key = h0 < key ? h0 : key;
                }
            } else {  // 2^31 <= p < 2^32
                for (int k = slice; k < n; k += S) {
                    const uint32_t x = xs[k];
                    const unsigned long long kk = (mul_add_mod64(A, B, x, p, inv_p) << 32) | x;
                    key = kk < key ? kk : key;
                }
            }
            k1 = k1 < k2 ? k1 : k2;
            k3 = k3 < key ? k3 : key;
            key = k1 < k3 ? k1 : k3;
        }
        for (int o = S / 2; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other < key ? other : key;
        }
        if (i < i_end && slice == 0) {
            const uint32_t arg = (uint32_t)key;
            if (out_dtype == MHB_OUT_I64) reinterpret_cast<long long*>(out)[set * n_hash + i] = (long long)arg;
            else reinterpret_cast<uint32_t*>(out)[set * n_hash + i] = arg;
        }
    }
    return flags;
}

__device__ __forceinline__ int check_ids(const uint32_t* xs, int n, uint64_t p) {
    int flags = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        if (xs[k] >= p) flags |= MHB_STATUS_ID_GE_PRIME;
    return flags;
}

// grid (hash slices, sets): block (x, s) computes hashes [x*kSmallSliceHashes, ...) of set s.
__global__ void __launch_bounds__(256) sign_small_kernel(int kind, const int64_t* indptr, const uint32_t* ids,
                                                        uint64_t a, uint64_t b, const uint32_t* ra,
                                                        const uint32_t* rb, uint64_t p, int32_t n_hash, void* out,
                                                        int32_t out_dtype, int32_t* status) {
    __shared__ uint32_t xs[kSmallSetMax];
    __shared__ int block_flags;
    if (threadIdx.x == 0) block_flags = 0;
    const int64_t set = blockIdx.y;
    const int64_t f0 = indptr[set] - indptr[0];
    const int n = (int)(indptr[set + 1] - indptr[set]);
    const int32_t i_begin = (int32_t)blockIdx.x * kSmallSliceHashes;
    const int32_t i_end = min(n_hash, i_begin + kSmallSliceHashes);
    int flags = n <= 0 ? MHB_STATUS_EMPTY_SET : 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) xs[k] = ids[f0 + k];
    __syncthreads();
    if (blockIdx.x == 0) flags |= check_ids(xs, n, p);
    flags |= small_set_hashes(xs, n, kind, a, b, ra, rb, p, n_hash, i_begin, i_end, out, out_dtype, set);
    if (flags) atomicOr(&block_flags, flags);  // (__syncthreads_or would only say "some flag")
    __syncthreads();
    if (threadIdx.x == 0) status[blockIdx.y * gridDim.x + blockIdx.x] = block_flags;  // one word per block
}

// ---- doorbell server: the per-set API without a kernel launch per call ----
//
// A per-set signature() call (the reference's own calling pattern, minhash.py:91-110,
// bench.py:97-102) is a few thousand visits, so the launch + stream sync of the small
// kernel dominate it.  Instead one block stays resident and polls a request word in
// mapped host memory.  The host packs the request (header | indptr | ids | a | b) into
// one mapped buffer and publishes {number, bytes} with one 64-bit release store; the
// block pulls the whole request into shared memory with 16-byte loads (one PCIe round
// trip for typical sets), computes, writes the signatures straight into mapped memory
// and publishes the number back after one system-scope fence
// (tools/doorbell_probe.cu measures each of these steps).  The block exits after
// MHB_DOORBELL_IDLE_US without a request, so device-wide syncs wait at most that
// long, and the host relaunches it on the next call.  MHB_DOORBELL=0 keeps the
// launched small kernel.
struct DoorbellReq {  // header of a packed request; then indptr[n_sets+1] | ids | a | b
    int32_t kind, n_hash, out_dtype, n_sets;
    uint64_t a, b, p;
    uint32_t ids_off, ra_off, rb_off, pad;  // byte offsets into the request
    unsigned long long out;                 // device address of the [n_sets, n_hash] output
};
static_assert(sizeof(DoorbellReq) % 16 == 0, "request header must keep 16-byte alignment");
constexpr uint32_t kDoorbellBytes = 40 * 1024;  // largest request the block stages in shared memory

struct alignas(64) Doorbell {  // mapped pinned control block
    unsigned long long post;      // host: (request bytes << 32) | request number (release)
    uint32_t done_seq;            // device: number of the last served request (release)
    uint32_t running;             // host sets 1 before a launch, the device clears it on exit
    uint32_t stop;                // host: exit now (release)
    unsigned long long trace[4];  // device, at each exit: summed load / compute / publish ns, requests
};

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kDoorbellThreads = 1024;

__global__ void __launch_bounds__(kDoorbellThreads, 1)
    doorbell_kernel(Doorbell* db, const uint4* req, int32_t* status, uint32_t served, uint64_t idle_ns) {
    __shared__ uint4 buf[kDoorbellBytes / 16];
    __shared__ uint32_t s_seq, s_bytes;
    __shared__ int s_go, block_flags;
    uint64_t last = global_ns();
    unsigned long long t_load = 0, t_compute = 0, t_publish = 0, n_served = 0;  // MHB_DOORBELL_TRACE
    for (;;) {
        if (threadIdx.x == 0) {
            int go = 0;
            unsigned long long post = 0;
            for (unsigned it = 0;; ++it) {
                post = ld_acquire_sys64(&db->post);
                if ((uint32_t)post != served) {
                    go = 1;
                    break;
                }
                if ((it & 15) == 15) {  // the stop word and the clock only now and then
                    if (ld_relaxed_sys(&db->stop) || global_ns() - last > idle_ns) break;
                }
            }
            if (!go) {
                db->trace[0] += t_load;
                db->trace[1] += t_compute;
                db->trace[2] += t_publish;
                db->trace[3] += n_served;
                st_release_sys(&db->running, 0u);  // the host relaunches for anything posted after this
            }
            s_go = go;
            s_seq = (uint32_t)post;
            s_bytes = (uint32_t)(post >> 32);
            block_flags = 0;
        }
        __syncthreads();
        if (!s_go) return;
        const unsigned long long tr0 = global_ns();
        const uint32_t n16 = s_bytes / 16;
        for (uint32_t k = threadIdx.x; k < n16; k += blockDim.x) buf[k] = __ldcv(req + k);
        __syncthreads();
        const DoorbellReq& rq = *reinterpret_cast<const DoorbellReq*>(buf);
        const char* base = reinterpret_cast<const char*>(buf);
        const int64_t* indptr = reinterpret_cast<const int64_t*>(base + sizeof(DoorbellReq));
        const uint32_t* ids = reinterpret_cast<const uint32_t*>(base + rq.ids_off);
        const uint32_t* ra = reinterpret_cast<const uint32_t*>(base + rq.ra_off);
        const uint32_t* rb = reinterpret_cast<const uint32_t*>(base + rq.rb_off);
        const unsigned long long tr1 = global_ns();
        int flags = 0;
        for (int set = 0; set < rq.n_sets; ++set) {
            const int64_t f0 = indptr[set] - indptr[0];
            const int n = (int)(indptr[set + 1] - indptr[set]);
            if (n <= 0) flags |= MHB_STATUS_EMPTY_SET;
            flags |= check_ids(ids + f0, n, rq.p);
            flags |= small_set_hashes(ids + f0, n, rq.kind, rq.a, rq.b, ra, rb, rq.p, rq.n_hash, 0, rq.n_hash,
                                      reinterpret_cast<void*>(rq.out), rq.out_dtype, set);
        }
        if (flags) atomicOr(&block_flags, flags);
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long tr2 = global_ns();
            t_load += tr1 - tr0;
            t_compute += tr2 - tr1;
            status[0] = block_flags;
            // the release (a system-scope fence + store) is cumulative over every thread's output
            // stores, which the barrier above ordered before it
            st_release_sys(&db->done_seq, s_seq);
            t_publish += global_ns() - tr2;
            ++n_served;
        }
        served = s_seq;
        last = global_ns();
        __syncthreads();  // buf and the s_* words are rewritten by the next request
    }
}

int grow(void** ptr, size_t* cap, size_t need) {
    if (*cap >= need && *ptr) return MHB_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    size_t want = need + need / 4 + 256;
    int rc = cuda_check(cudaMalloc(ptr, want), "cudaMalloc (host pipeline buffer)");
    if (rc) return rc;
    *cap = want;
    return MHB_OK;
}

struct Chunk {
    int64_t s0, s1;  // sets [s0, s1)
};

std::vector<Chunk> plan_chunks(const int64_t* indptr, int64_t n_sets, int32_t n_hash, size_t out_bytes) {
    // Cuts balanced by the bytes each chunk moves over PCIe (4 B per id in, n_hash
    // u32 entries + its indptr word out): ~16 chunks for large inputs, none smaller than
    // 16 MB, and rows bounded so the output chunk stays <= 256 MB.  Balancing on bytes
    // rather than ids alone also pipelines output-heavy batches (few sets, many hashes:
    // the reference's C6 timing workload, 500 sets x 100,000 hashes).
    static const int64_t n_chunks = [] {  // MHB_HOST_CHUNKS: tuning override
        const char* e = std::getenv("MHB_HOST_CHUNKS");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? (int64_t)v : (int64_t)16;
    }();
    const int64_t row_bytes = (int64_t)n_hash * 4 + 8;
    auto weight = [&](int64_t s) { return 4 * (indptr[s] - indptr[0]) + s * row_bytes; };  // monotone in s
    const int64_t target = std::max<int64_t>(weight(n_sets) / n_chunks, 16ll << 20);
    const int64_t max_rows = std::max<int64_t>(1, (int64_t)((256ull << 20) / ((size_t)n_hash * out_bytes)));
    std::vector<Chunk> out;
    int64_t s = 0;
    while (s < n_sets) {
        const int64_t goal = weight(s) + target;
        int64_t lo = s + 1, hi = std::min<int64_t>(n_sets, s + max_rows);  // largest e in [lo, hi] with weight(e) <= goal
        if (weight(hi) <= goal) {
            lo = hi;
        } else {
            while (lo < hi) {
                const int64_t mid = lo + (hi - lo + 1) / 2;
                if (weight(mid) <= goal) lo = mid;
                else hi = mid - 1;
            }
        }
        out.push_back({s, lo});
        s = lo;
    }
    return out;
}

}  // namespace

}  // namespace mhb

namespace mhb {
namespace {

bool small_batch(const int64_t* indptr, int64_t n_sets, int32_t n_hash, uint64_t prime) {
    if (n_sets > kSmallSets || n_sets * (int64_t)n_hash > kSmallEntries || prime >= (1ull << 32)) return false;
    if (indptr[n_sets] - indptr[0] > kSmallNnz) return false;
    for (int64_t s = 0; s < n_sets; ++s)
        if (indptr[s + 1] - indptr[s] > kSmallSetMax || indptr[s + 1] < indptr[s]) return false;
    return true;
}

bool doorbell_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MHB_DOORBELL");
        return !(e && e[0] == '0');
    }();
    return on;
}

uint64_t doorbell_idle_ns() {
    static const uint64_t ns = [] {
        const char* e = std::getenv("MHB_DOORBELL_IDLE_US");
        const long long v = e ? std::atoll(e) : 0;
        return (uint64_t)(v > 0 ? v : 1000) * 1000ull;
    }();
    return ns;
}

// Doorbell eligibility: the packed request fits the block's shared-memory stage, and the
// work suits one SM (<= 2^18 visits, ~15 us; <= 128 KB of output over PCIe from one SM).
// Returns the request bytes, or 0 for "launch sign_small_kernel instead".
uint32_t doorbell_request_bytes(int32_t kind, int64_t n_sets, int64_t nnz, int32_t n_hash, size_t out_bytes) {
    if ((uint64_t)nnz * (uint64_t)n_hash > (1ull << 18) || out_bytes > (128u << 10)) return 0u;
    auto up16 = [](uint64_t v) { return (v + 15) & ~15ull; };
    uint64_t bytes = sizeof(DoorbellReq) + up16((uint64_t)(n_sets + 1) * 8) + up16((uint64_t)nnz * 4);
    if (kind == KIND_RANDOM) bytes += 2 * up16((uint64_t)n_hash * 4);
    return bytes > kDoorbellBytes ? 0u : (uint32_t)bytes;
}

// Pack the request into the mapped request buffer, post it to the resident server block
// (launching one if none is running) and spin until it has been served.
int doorbell_call(SmallStage& sm, int32_t kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
                  uint64_t a, uint64_t b, const uint32_t* a_host, const uint32_t* b_host, uint64_t prime,
                  int32_t n_hash, void* out_dev, int32_t out_dtype, uint32_t bytes) {
    int rc;
    if (!sm.db) {
        if ((rc = cuda_check(cudaHostAlloc((void**)&sm.db, sizeof(Doorbell), cudaHostAllocMapped),
                             "cudaHostAlloc (doorbell)")))
            return rc;
        std::memset((void*)sm.db, 0, sizeof(Doorbell));
        if ((rc = cuda_check(cudaHostAlloc((void**)&sm.req, kDoorbellBytes, cudaHostAllocMapped),
                             "cudaHostAlloc (doorbell request)")))
            return rc;
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&sm.db_stream, cudaStreamNonBlocking), "doorbell stream")))
            return rc;
    }
    auto up16 = [](uint64_t v) { return (uint32_t)((v + 15) & ~15ull); };
    const int64_t nnz = indptr[n_sets] - indptr[0];
    DoorbellReq h{kind, n_hash, out_dtype, (int32_t)n_sets, a, b, prime, 0, 0, 0, 0,
                  (unsigned long long)reinterpret_cast<uintptr_t>(out_dev)};
    h.ids_off = (uint32_t)sizeof(DoorbellReq) + up16((uint64_t)(n_sets + 1) * 8);
    h.ra_off = h.ids_off + up16((uint64_t)nnz * 4);
    h.rb_off = h.ra_off + (kind == KIND_RANDOM ? up16((uint64_t)n_hash * 4) : 0);
    std::memcpy(sm.req, &h, sizeof h);
    std::memcpy(sm.req + sizeof h, indptr, (size_t)(n_sets + 1) * 8);
    if (nnz) std::memcpy(sm.req + h.ids_off, ids + indptr[0], (size_t)nnz * 4);
    if (kind == KIND_RANDOM) {
        std::memcpy(sm.req + h.ra_off, a_host, (size_t)n_hash * 4);
        std::memcpy(sm.req + h.rb_off, b_host, (size_t)n_hash * 4);
    }
    Doorbell* db = sm.db;
    const uint32_t seq = sm.seq + 1;
    // request bytes before the number (x86-64 stores are ordered; the release keeps the compiler honest)
    __atomic_store_n(&db->post, ((unsigned long long)bytes << 32) | seq, __ATOMIC_RELEASE);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0;; ++spin) {
        if (__atomic_load_n(&db->done_seq, __ATOMIC_ACQUIRE) == seq) break;
        if (__atomic_load_n(&db->running, __ATOMIC_ACQUIRE) == 0) {
            // no server (first call, or it idled out before seeing this request): launch one;
            // it serves everything numbered after `served` immediately
            if (__atomic_load_n(&db->done_seq, __ATOMIC_ACQUIRE) == seq) break;
            __atomic_store_n(&db->stop, 0u, __ATOMIC_RELEASE);
            __atomic_store_n(&db->running, 1u, __ATOMIC_RELEASE);
            doorbell_kernel<<<1, kDoorbellThreads, 0, sm.db_stream>>>(db, reinterpret_cast<const uint4*>(sm.req),
                                                                      sm.status, sm.seq, doorbell_idle_ns());
            if ((rc = cuda_check(cudaGetLastError(), "doorbell_kernel launch"))) {
                __atomic_store_n(&db->running, 0u, __ATOMIC_RELEASE);
                return rc;
            }
        }
        if ((spin & 1023) == 1023) {
            // a failed server (sticky CUDA error) or a wedged device must not spin forever
            const cudaError_t e = cudaStreamQuery(sm.db_stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_check(e, "doorbell_kernel");
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
                return set_error(MHB_ERR_CUDA, "doorbell request %u not served within 20 s", seq);
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    sm.seq = seq;
    return MHB_OK;
}

// Stop the server block (if running) and wait for it to exit.
void doorbell_stop(SmallStage& sm) {
    if (!sm.db) return;
    if (std::getenv("MHB_DOORBELL_TRACE")) {  // per-stage device time of the served requests
        const double n = (double)sm.db->trace[3];
        fprintf(stderr, "doorbell trace: %.0f requests, load %.2f us, compute %.2f us, publish %.2f us\n", n,
                sm.db->trace[0] / n / 1e3, sm.db->trace[1] / n / 1e3, sm.db->trace[2] / n / 1e3);
    }
    __atomic_store_n(&sm.db->stop, 1u, __ATOMIC_RELEASE);
    cudaStreamSynchronize(sm.db_stream);
    __atomic_store_n(&sm.db->running, 0u, __ATOMIC_RELEASE);
}

bool small_dev_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MHB_SMALL_DEV");
        return !(e && e[0] == '0');
    }();
    return on;
}

int grow_mapped(char** ptr, size_t* cap, size_t need, const char* what) {
    if (*cap >= need && *ptr) return MHB_OK;
    if (*ptr) cudaFreeHost(*ptr);
    *ptr = nullptr;
    *cap = 0;
    const size_t want = std::max<size_t>(need + need / 4, 1 << 20);
    int rc = cuda_check(cudaHostAlloc((void**)ptr, want, cudaHostAllocMapped), what);
    if (rc) return rc;
    *cap = want;
    return MHB_OK;
}

int sign_small(DeviceCache& dc, int32_t kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
               uint64_t a, uint64_t b, const uint32_t* a_host, const uint32_t* b_host, bool params_dev,
               uint64_t prime, int32_t n_hash, void* out, int32_t out_dtype, int32_t* status_host) {
    SmallStage& sm = dc.small;
    int rc;
    if (!sm.status) {
        if ((rc = cuda_check(cudaHostAlloc((void**)&sm.status, kSmallStatus * 4, cudaHostAllocMapped),
                             "cudaHostAlloc (small status)")))
            return rc;
    }
    const int64_t nnz = indptr[n_sets] - indptr[0];
    const size_t out_bytes = (size_t)n_sets * n_hash * (out_dtype == MHB_OUT_I64 ? 8 : 4);
    // A page-locked caller buffer is written by the kernel directly (UVA: the device address
    // of mapped host memory); the pointer query is paid only where a host copy would cost more.
    void* out_dev = nullptr;
    if (out_bytes >= (64u << 10) && is_pinned(out)) {
        if (cudaHostGetDevicePointer(&out_dev, out, 0) != cudaSuccess) {
            cudaGetLastError();
            out_dev = nullptr;
        }
    }
    if (!out_dev) {
        if ((rc = grow_mapped(&sm.out, &sm.out_cap, out_bytes, "cudaHostAlloc (small out)"))) return rc;
        out_dev = sm.out;
    }
    // (random-family parameters already on the device go to the launched kernel as they are)
    const uint32_t db_bytes = doorbell_enabled() && !params_dev
                                  ? doorbell_request_bytes(kind, n_sets, nnz, n_hash, out_bytes) : 0u;
    int64_t n_status = 1;  // words of sm.status the call wrote
    if (db_bytes) {
        if ((rc = doorbell_call(sm, kind, indptr, ids, n_sets, a, b, a_host, b_host, prime, n_hash, out_dev,
                                out_dtype, db_bytes)))
            return rc;
    } else {
        // Launched grid.  Wide outputs (>= 64 KB: the C6 shape, 100,000 hashes per set) go
        // through device memory with the copy engines on both sides -- one DMA of the packed
        // request in, one of the argmins out -- because hundreds of blocks reading and writing
        // mapped host memory directly cost 1.4x more (MHB_SMALL_DEV=0 keeps that path).
        auto up16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
        const bool stage_params = kind == KIND_RANDOM && !params_dev;
        const size_t ids_off = up16((size_t)(n_sets + 1) * 8), ra_off = ids_off + up16((size_t)nnz * 4);
        const size_t in_bytes = ra_off + (stage_params ? 2 * (size_t)n_hash * 4 : 0);
        if ((rc = grow_mapped(&sm.in, &sm.in_cap, in_bytes, "cudaHostAlloc (small in)"))) return rc;
        std::memcpy(sm.in, indptr, (n_sets + 1) * 8);
        if (nnz) std::memcpy(sm.in + ids_off, ids + indptr[0], nnz * 4);
        if (stage_params) {
            std::memcpy(sm.in + ra_off, a_host, n_hash * 4);
            std::memcpy(sm.in + ra_off + (size_t)n_hash * 4, b_host, n_hash * 4);
        }
        cudaStream_t st = dc.lanes[0].stream;
        const dim3 grid((unsigned)((n_hash + kSmallSliceHashes - 1) / kSmallSliceHashes), (unsigned)n_sets);
        n_status = (int64_t)grid.x * grid.y;
        const bool via_dev = out_bytes >= (64u << 10) && small_dev_enabled();
        char* base = sm.in;  // where the kernel reads the request
        void* kout = out_dev;
        int32_t* kstatus = sm.status;  // one plain store per block into mapped memory, either way
        if (via_dev) {
            const size_t out_off = up16(in_bytes);
            if ((rc = grow(&sm.dev, &sm.dev_cap, out_off + out_bytes))) return rc;
            base = static_cast<char*>(sm.dev);
            kout = base + out_off;
            if ((rc = cuda_check(cudaMemcpyAsync(base, sm.in, in_bytes, cudaMemcpyHostToDevice, st), "H2D small")))
                return rc;
        }
        const int64_t* ip = reinterpret_cast<const int64_t*>(base);
        const uint32_t* x = reinterpret_cast<const uint32_t*>(base + ids_off);
        const uint32_t* ra = stage_params ? reinterpret_cast<const uint32_t*>(base + ra_off) : a_host;
        const uint32_t* rb = stage_params ? ra + n_hash : b_host;
        sign_small_kernel<<<grid, 256, 0, st>>>(kind, ip, x, a, b, ra, rb, prime, n_hash, kout, out_dtype, kstatus);
        if ((rc = cuda_check(cudaGetLastError(), "sign_small_kernel launch"))) return rc;
        if (via_dev) {
            if ((rc = cuda_check(cudaMemcpyAsync(out_dev, kout, out_bytes, cudaMemcpyDeviceToHost, st), "D2H small")))
                return rc;
        }
        if ((rc = cuda_check(cudaStreamSynchronize(st), "sign_small_kernel"))) return rc;
    }
    if (out_dev == sm.out) {
        if (out_bytes >= (1u << 20)) host_copy_out(reinterpret_cast<const uint32_t*>(sm.out), out, out_bytes / 4, false);
        else std::memcpy(out, sm.out, out_bytes);
    }
    int32_t st_or = 0;
    for (int64_t s = 0; s < n_status; ++s) st_or |= sm.status[s];
    if (status_host) *status_host = st_or;
    return MHB_OK;
}

}  // namespace
}  // namespace mhb

using namespace mhb;

extern "C" int mhb_sign_csr_host(int32_t kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
                                 int64_t nnz, uint64_t a, uint64_t b, const uint32_t* a_host,
                                 const uint32_t* b_host, uint64_t prime, int32_t n_hash, void* out,
                                 int32_t out_dtype, int32_t* status_host, int32_t device) {
    clear_error();
    if (kind != KIND_ITERATIVE && kind != KIND_RANDOM) return set_error(MHB_ERR_INVALID, "unknown kind %d", kind);
    if (n_sets < 0) return set_error(MHB_ERR_INVALID, "n_sets must be >= 0");
    if (status_host) *status_host = 0;
    if (n_sets == 0) return MHB_OK;
    if (!indptr || !out || (nnz > 0 && !ids)) return set_error(MHB_ERR_INVALID, "null host pointer");
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function, got %d", n_hash);
    if (indptr[n_sets] - indptr[0] > nnz) return set_error(MHB_ERR_INVALID, "indptr exceeds nnz");
    if (out_dtype != MHB_OUT_U32 && out_dtype != MHB_OUT_I64)
        return set_error(MHB_ERR_INVALID, "unknown out_dtype %d", out_dtype);
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) {  // -1: the calling thread's current device
        cudaGetLastError();
        return set_error(MHB_ERR_CUDA, "no current CUDA device");
    }
    if (device >= 64) return set_error(MHB_ERR_INVALID, "bad device %d", device);
    const size_t out_bytes = out_dtype == MHB_OUT_I64 ? 8 : 4;

    std::lock_guard<std::mutex> lock(g_mu);
    struct DeviceGuard {  // restores the caller's current device on every return path
        int prev = 0;
        bool moved = false;
        DeviceGuard() { cudaGetDevice(&prev); }
        ~DeviceGuard() {
            if (moved) cudaSetDevice(prev);
        }
    } guard;
    int rc = MHB_OK;
    if (guard.prev != device) {
        guard.moved = true;
        if ((rc = cuda_check(cudaSetDevice(device), "cudaSetDevice"))) return rc;
    }
    DeviceCache& dc = g_cache[device];
    if (!dc.init) {
        for (auto& ln : dc.lanes) {
            rc = cuda_check(cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking), "stream create");
            if (rc) return rc;
            rc = cuda_check(cudaEventCreateWithFlags(&ln.done, cudaEventDisableTiming), "event create");
            if (rc) return rc;
        }
        rc = cuda_check(cudaMalloc((void**)&dc.status, kMaxChunks * sizeof(int32_t)), "cudaMalloc status");
        if (rc) return rc;
        dc.init = true;
    }
    if (kind == KIND_RANDOM && (!a_host || !b_host)) return set_error(MHB_ERR_INVALID, "random family needs a and b");
    // random-family a/b may also be device arrays (UVA): used in place, no staging
    const bool params_dev = kind == KIND_RANDOM && is_device_ptr(a_host) && is_device_ptr(b_host);
    if (small_batch(indptr, n_sets, n_hash, prime)) {
        if ((rc = check_sign_params(kind, a, b, true, prime, n_hash))) return rc;
        return sign_small(dc, kind, indptr, ids, n_sets, a, b, a_host, b_host, params_dev, prime, n_hash, out,
                          out_dtype, status_host);
    }
    const uint32_t* ra_dev = dc.ra;
    const uint32_t* rb_dev = dc.rb;
    if (params_dev) {
        ra_dev = a_host;
        rb_dev = b_host;
    } else if (kind == KIND_RANDOM) {
        if ((rc = grow((void**)&dc.ra, &dc.ra_cap, (size_t)n_hash * 4))) return rc;
        if ((rc = grow((void**)&dc.rb, &dc.rb_cap, (size_t)n_hash * 4))) return rc;
        cudaStream_t s0 = dc.lanes[0].stream;
        if ((rc = cuda_check(cudaMemcpyAsync(dc.ra, a_host, (size_t)n_hash * 4, cudaMemcpyHostToDevice, s0), "H2D a")))
            return rc;
        if ((rc = cuda_check(cudaMemcpyAsync(dc.rb, b_host, (size_t)n_hash * 4, cudaMemcpyHostToDevice, s0), "H2D b")))
            return rc;
        if ((rc = cuda_check(cudaStreamSynchronize(s0), "sync params"))) return rc;
        ra_dev = dc.ra;
        rb_dev = dc.rb;
    }

    const std::vector<Chunk> chunks = plan_chunks(indptr, n_sets, n_hash, out_bytes);
    if (chunks.size() > (size_t)kMaxChunks) return set_error(MHB_ERR_INVALID, "batch needs more than %d chunks", kMaxChunks);
    int32_t status_acc = 0;
    // Pageable caller buffers would make every cudaMemcpyAsync synchronous (staged by the
    // driver).  So: ids from pageable memory are copied into a pinned lane buffer by the
    // host pool before their H2D; for pageable output the kernels write uint32, the D2H
    // lands in a pinned lane buffer, and the pool copies (or widens to int64: half the
    // PCIe bytes) into the caller's array once the lane drains -- overlapped with the
    // transfers of the other lanes.  Pinned output keeps the direct D2H.
    // Pinned int64 output is staged the same way: uint32 over PCIe plus a streaming-store
    // widening on the host beats the DMA writing twice the bytes (37 vs 42 ms on cfg2;
    // MHB_DIRECT_I64=1 keeps the direct int64 D2H).
    const bool stage_out = !is_pinned(out) || (out_dtype == MHB_OUT_I64 && !direct_i64());
    const bool widen = stage_out && out_dtype == MHB_OUT_I64;
    const bool stage_in = nnz > 0 && !is_pinned(ids);
    auto drain = [&](Lane& ln) {
        if (ln.pend_s0 >= 0) {
            host_copy_out(ln.stage_out, static_cast<char*>(out) + (size_t)ln.pend_s0 * n_hash * out_bytes,
                          ln.pend_rows * (int64_t)n_hash, widen);
            ln.pend_s0 = -1;
        }
    };

    for (size_t c = 0; c < chunks.size(); ++c) {
        Lane& ln = dc.lanes[c % kLanes];
        const int64_t s0 = chunks[c].s0, s1 = chunks[c].s1, rows = s1 - s0;
        const int64_t id0 = indptr[s0], id1 = indptr[s1];
        const int64_t cnnz = id1 - id0;
        if (c >= (size_t)kLanes) {
            // the lane's previous chunk must have drained before its buffers are reused
            if ((rc = cuda_check(cudaEventSynchronize(ln.done), "lane sync"))) return rc;
            drain(ln);
        }
        if ((rc = grow((void**)&ln.indptr, &ln.indptr_cap, (size_t)(rows + 1) * sizeof(int64_t)))) return rc;
        if ((rc = grow((void**)&ln.ids, &ln.ids_cap, (size_t)std::max<int64_t>(cnnz, 1) * sizeof(uint32_t))))
            return rc;
        const size_t dev_out_bytes = (size_t)rows * n_hash * (stage_out ? 4 : out_bytes);
        if ((rc = grow(&ln.out, &ln.out_cap, dev_out_bytes))) return rc;
        const size_t wsb = mhb_sign_workspace_bytes(rows, cnnz, n_hash);
        if ((rc = grow(&ln.ws, &ln.ws_cap, wsb))) return rc;

        if ((rc = cuda_check(cudaMemcpyAsync(ln.indptr, indptr + s0, (size_t)(rows + 1) * sizeof(int64_t),
                                             cudaMemcpyHostToDevice, ln.stream), "H2D indptr")))
            return rc;
        const uint32_t* id_src = ids + id0;
        if (stage_in && cnnz > 0) {
            if ((rc = grow_pinned((void**)&ln.stage_ids, &ln.stage_ids_cap, (size_t)cnnz * 4))) return rc;
            host_copy_in(ids + id0, ln.stage_ids, cnnz);
            id_src = ln.stage_ids;
        }
        if (cnnz > 0 &&
            (rc = cuda_check(cudaMemcpyAsync(ln.ids, id_src, (size_t)cnnz * sizeof(uint32_t),
                                             cudaMemcpyHostToDevice, ln.stream), "H2D ids")))
            return rc;
        // Rebase the chunk's offsets onto its own ids buffer (ids[0..cnnz) is what the kernels may read).
        if (id0 != 0) {
            const int64_t nb = std::min<int64_t>((rows + 1 + 255) / 256, 1024);
            rebase_indptr_kernel<<<(unsigned)nb, 256, 0, ln.stream>>>(ln.indptr, rows + 1, id0);
            if ((rc = cuda_check(cudaGetLastError(), "rebase_indptr launch"))) return rc;
        }
        rc = launch_sign(kind, ln.indptr, ln.ids, rows, cnnz, a, b, ra_dev, rb_dev, prime, n_hash, ln.out,
                         stage_out ? MHB_OUT_U32 : out_dtype, dc.status + c, ln.ws, ln.ws_cap, ln.stream);
        if (rc) return rc;
        if (stage_out) {
            if ((rc = grow_pinned((void**)&ln.stage_out, &ln.stage_out_cap, dev_out_bytes))) return rc;
            if ((rc = cuda_check(cudaMemcpyAsync(ln.stage_out, ln.out, dev_out_bytes, cudaMemcpyDeviceToHost,
                                                 ln.stream), "D2H out (staged)")))
                return rc;
            ln.pend_s0 = s0;
            ln.pend_rows = rows;
        } else if ((rc = cuda_check(cudaMemcpyAsync(static_cast<char*>(out) + (size_t)s0 * n_hash * out_bytes, ln.out,
                                                    dev_out_bytes, cudaMemcpyDeviceToHost, ln.stream),
                                    "D2H out"))) {
            return rc;
        }
        if ((rc = cuda_check(cudaEventRecord(ln.done, ln.stream), "event record"))) return rc;
    }
    for (int l = 0; l < kLanes && (size_t)l < chunks.size(); ++l) {
        if ((rc = cuda_check(cudaStreamSynchronize(dc.lanes[l].stream), "final sync"))) return rc;
        drain(dc.lanes[l]);
    }
    std::vector<int32_t> st(chunks.size());
    if ((rc = cuda_check(cudaMemcpy(st.data(), dc.status, chunks.size() * sizeof(int32_t), cudaMemcpyDeviceToHost),
                         "status read")))
        return rc;
    for (int32_t v : st) status_acc |= v;
    if (status_host) *status_host = status_acc;
    return MHB_OK;
}

extern "C" void mhb_host_release(void) {
    std::lock_guard<std::mutex> lock(g_mu);
    for (int d = 0; d < 64; ++d) {
        DeviceCache& dc = g_cache[d];
        if (!dc.init) continue;
        cudaSetDevice(d);
        for (auto& ln : dc.lanes) {
            cudaStreamSynchronize(ln.stream);
            cudaFree(ln.indptr);
            cudaFree(ln.ids);
            cudaFree(ln.out);
            cudaFree(ln.ws);
            if (ln.stage_ids) cudaFreeHost(ln.stage_ids);
            if (ln.stage_out) cudaFreeHost(ln.stage_out);
            cudaEventDestroy(ln.done);
            cudaStreamDestroy(ln.stream);
            ln = Lane{};
        }
        cudaFree(dc.ra);
        cudaFree(dc.rb);
        cudaFree(dc.status);
        doorbell_stop(dc.small);
        if (dc.small.db_stream) cudaStreamDestroy(dc.small.db_stream);
        if (dc.small.db) cudaFreeHost(dc.small.db);
        if (dc.small.req) cudaFreeHost(dc.small.req);
        if (dc.small.dev) cudaFree(dc.small.dev);
        if (dc.small.in) cudaFreeHost(dc.small.in);
        if (dc.small.out) cudaFreeHost(dc.small.out);
        if (dc.small.status) cudaFreeHost(dc.small.status);
        dc = DeviceCache{};
    }
}
