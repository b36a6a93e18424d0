// small.cu -- small batches of the host-buffer entry (mhb_sign_csr_host): the per-set
// reference API (signature() on one FeatureSet, minhash.py:91-110) and the reference's
// own per-document timing loop (run_timing, bench.py:97-102; C6: one set x 100,000
// hashes per call).  See host_internal.h for the routing constants.
//
//  - doorbell_kernel: one resident block polling a request word in mapped host memory
//    serves light requests without a launch (tools/doorbell_probe.cu for the protocol).
//  - sign_small_kernel: one launch over (hash slice, set) blocks for heavier requests;
//    wide outputs go through device memory with one DMA each way.
// Both compute every (set, hash) argmin exactly (small_set_hashes), u32 Shoup lanes for
// p < 2^31 and 64-bit residues up to 2^32.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.h"
#include "host_internal.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

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

namespace {

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
// and publishes the number back with one system-scope release (DoorbellReq / Doorbell
// above; tools/doorbell_probe.cu measures each of these steps).  The block exits after
// MHB_DOORBELL_IDLE_US without a request, so device-wide syncs wait at most that
// long, and the host relaunches it on the next call.  MHB_DOORBELL=0 keeps the
// launched small kernel.
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

}  // namespace

bool small_batch(const int64_t* indptr, int64_t n_sets, int32_t n_hash, uint64_t prime) {
    if (n_sets > kSmallSets || n_sets * (int64_t)n_hash > kSmallEntries || prime >= (1ull << 32)) return false;
    if (indptr[n_sets] - indptr[0] > kSmallNnz) return false;
    for (int64_t s = 0; s < n_sets; ++s)
        if (indptr[s + 1] - indptr[s] > kSmallSetMax || indptr[s + 1] < indptr[s]) return false;
    return true;
}

int sign_small(SmallStage& sm, cudaStream_t stream, int32_t kind, const int64_t* indptr, const uint32_t* ids,
               int64_t n_sets, uint64_t a, uint64_t b, const uint32_t* a_host, const uint32_t* b_host,
               bool params_dev, uint64_t prime, int32_t n_hash, void* out, int32_t out_dtype,
               int32_t* status_host) {
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
        cudaStream_t st = stream;
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
        if (out_bytes >= (256u << 10))  // 64 KB per worker: a wide per-set result is ~1 MB
            host_copy_out(reinterpret_cast<const uint32_t*>(sm.out), out, out_bytes / 4, false, 1 << 14);
        else std::memcpy(out, sm.out, out_bytes);
    }
    int32_t st_or = 0;
    for (int64_t s = 0; s < n_status; ++s) st_or |= sm.status[s];
    if (status_host) *status_host = st_or;
    return MHB_OK;
}


void small_release(SmallStage& sm) {
    doorbell_stop(sm);
    if (sm.db_stream) cudaStreamDestroy(sm.db_stream);
    if (sm.db) cudaFreeHost(sm.db);
    if (sm.req) cudaFreeHost(sm.req);
    if (sm.dev) cudaFree(sm.dev);
    if (sm.in) cudaFreeHost(sm.in);
    if (sm.out) cudaFreeHost(sm.out);
    if (sm.status) cudaFreeHost(sm.status);
    sm = SmallStage{};
}

}  // namespace mhb
