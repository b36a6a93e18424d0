// host.cu -- host-buffer entry point: chunked, copy/compute-overlapped signing.
//
// The reference's callers hand numpy arrays to the signing loop and get numpy
// arrays back (minhash.py:91-110, bench.py:97-102).  mhb_sign_csr_host is the
// native equivalent for a whole CSR batch living in host memory: the sets are
// cut into nnz-balanced chunks; each chunk goes H2D -> sign kernels -> D2H on
// one of 4 stream lanes, so the copy engines (both directions) and the SMs
// work on different chunks at the same time.  Device buffers are cached per
// device between calls (mhb_host_release frees them).  Small batches (the per-set
// reference API) take the paths of small.cu instead.
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
#include "host_internal.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

// ---- host-memory helpers (also used by small.cu, declared in host_internal.h) ----
namespace {

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
    // fn(part) for part in [0, parts), spread over the pool and the caller.  Callers are
    // serialised (one job at a time).
    void run(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1 || th_.empty()) {
            for (int k = 0; k < parts; ++k) fn(k);
            return;
        }
        std::lock_guard<std::mutex> serial(run_mu_);
        uint64_t gen;
        {
            std::lock_guard<std::mutex> l(m_);
            gen = ++gen_;
            fn_ = &fn;
            parts_ = parts;
            left_ = parts;
            // claims carry the job generation in the high word: a worker still holding the
            // previous job can never take (and so never run or double-count) a part of this one
            claim_.store(gen << 32);
        }
        cv_.notify_all();
        work(gen, &fn, parts);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [this] { return left_ == 0; });
        fn_ = nullptr;
    }
    int width() const { return (int)th_.size() + 1; }

  private:
    // Claim parts of job `gen` until none is left or a newer job replaced it.  The claim is
    // a CAS on (gen << 32 | next part), so it fails instead of consuming a part of another job.
    void work(uint64_t gen, const std::function<void(int)>* fn, int parts) {
        for (;;) {
            uint64_t v = claim_.load();
            int k;
            for (;;) {
                if ((v >> 32) != (gen & 0xffffffffull)) return;
                k = (int)(v & 0xffffffffull);
                if (k >= parts) return;
                if (claim_.compare_exchange_weak(v, v + 1)) break;
            }
            (*fn)(k);
            std::lock_guard<std::mutex> l(m_);
            if (--left_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            uint64_t gen;
            const std::function<void(int)>* fn;
            int parts;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen = gen_;
                fn = fn_;  // the job of generation `gen` (valid until its parts are all done)
                parts = parts_;
            }
            if (fn) work(gen, fn, parts);
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, run_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int parts_ = 0, left_ = 0;
    std::atomic<uint64_t> claim_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

HostPool& host_pool() {
    static HostPool pool;
    return pool;
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

}  // namespace

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

// Parallel copy (u32 -> u32, or u32 -> int64 widening) of `n` elements.
void host_copy_out(const uint32_t* src, void* dst, int64_t n, bool widen, int64_t part_elems) {
    HostPool& pool = host_pool();
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool.width() * 2, n / part_elems));
    const bool nt = host_nt();
    pool.run(parts, [&](int k) {
        const int64_t lo = n * k / parts, hi = n * (k + 1) / parts;
        char* d = static_cast<char*>(dst) + (size_t)lo * (widen ? 8 : 4);
        copy_span(src + lo, d, hi - lo, widen, nt);
    });
}

// ---- the chunked pipeline ----
namespace {

constexpr int kMaxLanes = 8;

// Stream lanes in use (MHB_HOST_LANES, 2..8; default 4): chunk c runs on lane c % lanes,
// whose previous chunk must have drained before its buffers are reused.
int host_lanes() {
    static const int n = [] {
        const char* e = std::getenv("MHB_HOST_LANES");
        const int v = e ? std::atoi(e) : 4;
        return v < 2 ? 2 : (v > kMaxLanes ? kMaxLanes : v);
    }();
    return n;
}
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

void host_copy_in(const uint32_t* src, uint32_t* dst, int64_t n) {
    HostPool& pool = host_pool();
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool.width() * 2, n >> 18));
    const bool nt = host_nt();
    pool.run(parts, [&](int k) {
        const int64_t lo = n * k / parts, hi = n * (k + 1) / parts;
        copy_span(src + lo, dst + lo, hi - lo, false, nt);
    });
}

struct DeviceCache {
    bool init = false;
    SmallStage small;
    Lane lanes[kMaxLanes];
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
    // ids are read at the absolute offsets indptr[s]: they must lie in [0, nnz] and never decrease
    if (indptr[0] < 0 || indptr[n_sets] > nnz)
        return set_error(MHB_ERR_INVALID, "indptr must satisfy 0 <= indptr[0] and indptr[n_sets] <= nnz");
    for (int64_t s = 0; s < n_sets; ++s)
        if (indptr[s + 1] < indptr[s]) return set_error(MHB_ERR_INVALID, "indptr decreases at set %lld", (long long)s);
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
        return sign_small(dc.small, dc.lanes[0].stream, kind, indptr, ids, n_sets, a, b, a_host, b_host, params_dev,
                          prime, n_hash, out, out_dtype, status_host);
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
    const int n_lanes = host_lanes();
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
    // Any early return below leaves no work behind: every lane is synchronised (its D2H
    // into the caller's buffers has finished) and its staged chunk is forgotten, so a later
    // call never drains this call's rows into its own output.
    struct LaneReset {
        DeviceCache& dc;
        int n;
        bool ok = false;
        ~LaneReset() {
            if (ok) return;
            for (int l = 0; l < n; ++l) {
                cudaStreamSynchronize(dc.lanes[l].stream);
                dc.lanes[l].pend_s0 = -1;
            }
            cudaGetLastError();
        }
    } reset{dc, n_lanes};
    for (int l = 0; l < kMaxLanes; ++l) dc.lanes[l].pend_s0 = -1;

    for (size_t c = 0; c < chunks.size(); ++c) {
        Lane& ln = dc.lanes[c % (size_t)n_lanes];
        const int64_t s0 = chunks[c].s0, s1 = chunks[c].s1, rows = s1 - s0;
        const int64_t id0 = indptr[s0], id1 = indptr[s1];
        const int64_t cnnz = id1 - id0;
        if (c >= (size_t)n_lanes) {
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
    for (int l = 0; l < n_lanes && (size_t)l < chunks.size(); ++l) {
        if ((rc = cuda_check(cudaStreamSynchronize(dc.lanes[l].stream), "final sync"))) return rc;
        drain(dc.lanes[l]);
    }
    std::vector<int32_t> st(chunks.size());
    if ((rc = cuda_check(cudaMemcpy(st.data(), dc.status, chunks.size() * sizeof(int32_t), cudaMemcpyDeviceToHost),
                         "status read")))
        return rc;
    for (int32_t v : st) status_acc |= v;
    if (status_host) *status_host = status_acc;
    reset.ok = true;
    return MHB_OK;
}

extern "C" int mhb_host_pool_selftest(int64_t jobs, uint64_t seed, int32_t threads, int64_t* bad) {
    clear_error();
    if (!bad || jobs < 0 || threads < 1 || threads > 64) return set_error(MHB_ERR_INVALID, "bad arguments");
    std::atomic<int64_t> wrong{0};
    auto caller = [&](int t) {
        uint64_t s = seed * 6364136223846793005ull + (uint64_t)t * 1442695040888963407ull + 1;
        std::vector<std::atomic<int>> hits(64);
        for (int64_t j = t; j < jobs; j += threads) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            const int parts = 2 + (int)((s >> 33) % 63);
            for (int k = 0; k < parts; ++k) hits[k].store(0);
            const int spin = (int)((s >> 20) & 255);
            host_pool().run(parts, [&](int k) {
                volatile int x = 0;  // uneven part lengths: workers finish at different times
                for (int i = 0; i < spin * (k & 3); ++i) x = x + i;
                hits[k].fetch_add(1);
            });
            for (int k = 0; k < parts; ++k)
                if (hits[k].load() != 1) wrong.fetch_add(1);
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < threads; ++t) th.emplace_back(caller, t);
    caller(0);
    for (auto& x : th) x.join();
    *bad = wrong.load();
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
        small_release(dc.small);
        dc = DeviceCache{};
    }
}
