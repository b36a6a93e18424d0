// sign.cu -- MinHash signatures over CSR sets on sm_100a (both hash families).
//
// Reference semantics (arXiv 1401.6124 reference package `minhashlab`):
//   sign_iterative  kernels.py:44-73   h_i(x) = ((a+i)x + i*b) mod p, walked as
//                                      h <- h + (x+b) mod p with one conditional subtract
//   sign_random     kernels.py:21-41   h_i(x) = (a_i x + b_i) mod p
//   output          minhash.py:91-110  argmin feature id per hash index
//
// Design (DESIGN.md has the numbers):
//  * Plan (3 small kernels): sets are cut into virtual sets of <= kChunk features
//    and counting-sorted by size, largest first.
//  * Main kernel (persistent, dynamic work counter): a warp takes a group of F
//    consecutive virtual sets -- equal sizes, thanks to the sort -- one per slice.
//    Its 32 threads are G lane groups x F slices (G*F = 32): thread (g,f) keeps the
//    running minima of hash lanes i0..i0+K-1 (i0 = g*K) of set f in registers and
//    walks that set's features two at a time.  No cross-thread combine is needed
//    and a group wastes almost nothing at its end.
//  * Per (thread, feature): one Shoup multiply gives h_{i0}(x) = A_{i0} x + B_{i0};
//    then the iterative walk costs IADD + VIADDMNMX + 1/2 VIMNMX3 per visit, with a
//    two-lane lookahead that halves the dependent chain (tools/visit_probe.cu).
//    The random family costs IMAD.HI + 2 IMAD + 2 VIADDMNMX + 1/2 VIMNMX3 per visit.
//  * Only the min HASH VALUE is tracked.  Every member is a bijection on [0,p)
//    (families.py:82,141; test_families.py:178-186), so the argmin is recovered
//    exactly once per entry: x = (h - B_i) * A_i^{-1} mod p.
//  * Sets longer than kChunk merge their chunks with atomicMin on the output row;
//    a finalize pass inverts those rows.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <mutex>

#include "bandhash.cuh"
#include "common.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

// ----------------------------------------------------------------------------
// Geometry and workspace
// ----------------------------------------------------------------------------

static int next_pow2(int v) {
    int r = 1;
    while (r < v) r <<= 1;
    return r;
}

static int default_lanes(int kind, int32_t n_hash) {
    if (kind == KIND_ITERATIVE) return n_hash >= 128 ? 64 : n_hash >= 32 ? 32 : n_hash >= 16 ? 16 : 8;
    return n_hash >= 16 ? 16 : 8;  // 3 constants + 1 minimum per lane in registers
}

Geometry choose_geometry(int kind, int32_t n_hash, int K) {
    Geometry g{};
    if (K <= 0) K = default_lanes(kind, n_hash);
    int lg = (n_hash + K - 1) / K;
    if (lg <= 32) {
        g.G = next_pow2(lg);
        g.n_super = 1;
    } else {
        g.G = 32;
        g.n_super = (n_hash + 32 * K - 1) / (32 * K);
    }
    g.K = K;
    g.F = 32 / g.G;
    g.log2F = 0;
    while ((1 << g.log2F) < g.F) ++g.log2F;
    g.L = g.G * K;
    g.n_tot = (int64_t)g.n_super * g.L;
    return g;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Lanes per thread for this batch.  The default K amortises each feature's start hash
// over many lanes, but a small batch then has too few work items (warps) to fill the
// SMs: cfg1 (10,000 sets, N = 128) gives 625 warps at K = 64 for 148 SMs x 16 warps.
// Iterative family: take the K (64, 32, 16, 8: more lane groups per set, so more warps)
// with the fewest waves x per-item work.  MHB_SIGN_K forces K (tuning).
constexpr int64_t kSmallPlanSets = 1 << 14;  // = kSmallPlan (batches signed by the one-launch plan)

static int pick_lanes(int kind, int32_t n_hash, int64_t n_sets, int sms, bool fixed) {
    static const int forced = [] {
        const char* e = std::getenv("MHB_SIGN_K");
        return e ? std::atoi(e) : 0;
    }();
    const int K0 = default_lanes(kind, n_hash);
    if (forced == 8 || forced == 16 || (kind == KIND_ITERATIVE && (forced == 32 || forced == 64)))
        return fixed ? K0 : forced;
    if (fixed || kind != KIND_ITERATIVE) return K0;
    // cost(K) ~ waves of items x per-item work: a thread's round costs ~2.5 K + 14
    // instructions (the walk plus the per-feature start hash, steps and loads)
    const int64_t slots = (int64_t)sms * 2 * (kBlock / 32);  // one wave of warp slots (2 CTAs/SM)
    int best = K0;
    double best_cost = -1.0;
    for (int K = K0; K >= 8; K /= 2) {
        const Geometry g = choose_geometry(kind, n_hash, K);
        const int64_t items = (n_sets + g.F - 1) / g.F * g.n_super;
        // small batches (one-launch plan, unsorted): whole waves; large batches (sorted,
        // dynamic counter): fractional waves plus half a wave of tail (cfg3 50k-set
        // shards: K = 64 at 5.3 waves beats K = 32 at 10.6)
        const double waves = n_sets <= kSmallPlanSets ? (double)((items + slots - 1) / slots)
                                                       : (double)items / (double)slots + 0.5;
        const double cost = waves * (5 * K + 28);
        if (best_cost < 0 || cost < best_cost) {
            best = K;
            best_cost = cost;
        }
    }
    return best;
}

static int forced_chunk() {
    static const int forced = [] {
        const char* e = std::getenv("MHB_CHUNK");
        const int v = e ? std::atoi(e) : 0;
        return (v == 256 || v == 512 || v == 1024) ? v : 0;
    }();
    return forced;
}

constexpr double kChunkVisits1024 = 34359738368.0;  // 2^35 visits and up: chunk 1024
constexpr double kChunkVisits512 = 8589934592.0;    // 2^33 visits and up: chunk 512, else 256

int choose_chunk(int64_t n_sets, int64_t nnz, int32_t n_hash) {
    if (const int forced = forced_chunk()) return forced;
    // A virtual set is one slice's item; the descending-size schedule starts the largest
    // first, but a few of them landing on one SMSP set the kernel's tail once they are a
    // sizeable share of an SMSP's work.  So the chunk shrinks with the batch's visits
    // N * nnz, but never below ~1.25x the mean set, so typical sets are not split (each
    // split set pays N merge atomics and a finalize pass).  tools/scaling_projection.py
    // (cfg2 shards, ms per shard at 1024 / 512 / 256): 197M ids 4.81 / 4.96 / 5.35,
    // 99M 2.62 / 2.51 / 2.70, 49M 1.56 / 1.35 / 1.41, 25M 1.25 / 0.85 / 0.77; cfg3
    // (Poisson(300) sets) 0.89 / 0.89 / 1.32 at 15M ids.
    const double visits = (double)(nnz > 0 ? nnz : 0) * (double)(n_hash > 0 ? n_hash : 1);
    int chunk = visits >= kChunkVisits1024 ? 1024 : visits >= kChunkVisits512 ? 512 : 256;
    const double mean = n_sets > 0 ? (double)nnz / (double)n_sets : 0.0;
    while (chunk < kChunk && chunk < 1.25 * mean) chunk *= 2;
    return chunk;
}

// Upper bound on the extra virtual sets (chunks beyond each set's first) of ANY batch
// with at most `nnz` ids: the max over nnz' <= nnz of nnz' / chunk(nnz').  It is
// monotone in nnz, so a workspace sized for a batch also fits every smaller one (the
// chunk shrinks with the batch, so nnz / chunk alone is not).
static int64_t extra_vsets_bound(int64_t nnz, int32_t n_hash) {
    if (nnz <= 0) return 0;
    if (const int forced = forced_chunk()) return nnz / forced;
    const double n = n_hash > 0 ? (double)n_hash : 1.0;
    const int64_t t512 = (int64_t)(kChunkVisits512 / n), t1024 = (int64_t)(kChunkVisits1024 / n);
    int64_t b = nnz / 1024;
    b = std::max<int64_t>(b, std::min<int64_t>(nnz, t1024) / 512);
    b = std::max<int64_t>(b, std::min<int64_t>(nnz, t512) / 256);
    return b;
}

WorkspaceLayout workspace_layout(int64_t n_sets, int64_t nnz, int32_t n_hash) {
    // Both families and every lane count share one layout; size for the largest lane table.
    int64_t n_tot = 0;
    for (int K = 8; K <= 64; K *= 2)
        for (int kind = 0; kind < 2; ++kind) {
            const Geometry g = choose_geometry(kind, n_hash, K);
            if (g.n_tot > n_tot) n_tot = g.n_tot;
        }
    int64_t nnz_pos = nnz > 0 ? nnz : 0;
    int64_t sets = n_sets > 0 ? n_sets : 0;
    // every long set has at least one extra chunk
    const int64_t extra = extra_vsets_bound(nnz_pos, n_hash);
    int64_t max_big = extra;
    if (max_big > sets) max_big = sets;
    int64_t max_vsets = sets + extra;

    WorkspaceLayout w{};
    size_t off = 0;
    w.sched = off;  off = align_up(off + sizeof(Sched), 256);
    w.hist = off;   off = align_up(off + 2 * kChunk * sizeof(unsigned), 256);
    w.tab = off;    off = align_up(off + (size_t)n_tot * sizeof(LaneTab), 256);
    w.inv = off;    off = align_up(off + (size_t)n_tot * sizeof(InvTab), 256);
    w.big = off;    off = align_up(off + (size_t)(max_big > 0 ? max_big : 1) * sizeof(int64_t), 256);
    w.vsets = off;  off = align_up(off + (size_t)(max_vsets > 0 ? max_vsets : 1) * sizeof(VSet), 256);
    w.total = off;
    return w;
}

// ----------------------------------------------------------------------------
// Plan: lane tables, size histogram of virtual sets, long-set bookkeeping
// ----------------------------------------------------------------------------

// floor(w * 2^32 / p) for w < p < 2^31 without the 64-bit division (a long emulated
// sequence): a double-precision estimate, corrected against the exact 64-bit remainder.
__device__ __forceinline__ uint32_t companion_fast(uint32_t w, uint32_t p) {
    uint32_t q = (uint32_t)(((double)w * 4294967296.0) / (double)p);
    int64_t r = (int64_t)((uint64_t)w << 32) - (int64_t)q * (int64_t)p;
    while (r < 0) { --q; r += p; }
    while (r >= (int64_t)p) { ++q; r -= p; }
    return q;
}

// Lane i's tables: the start-hash constants (A, Shoup(A), B) and the argmin recovery
// (B, A^{-1}, Shoup(A^{-1})).  All 32-bit arithmetic (p < 2^31).
__device__ __forceinline__ void fill_lane_tables(const SignArgs& A, int64_t i) {
    const uint32_t p = A.p;
    uint32_t w, c;
    if (A.kind == KIND_ITERATIVE) {
        // member i: multiplier a+i, offset i*b (families.py:124-131)
        w = (uint32_t)(((uint32_t)A.ia + (uint32_t)(i % p)) % p);  // a < p < 2^31: no overflow
        if (w == 0) w = 1;  // only reachable on padded lanes i >= n_hash
        c = reduce_once(shoup_lazy(A.b, companion_fast(A.b, p), (uint32_t)(i % p), p), p);
    } else if (i < A.n_hash) {
        w = A.ra[i];
        c = A.rb[i];
        if (w == 0 || w >= p || c >= p) {
            if (A.status) atomicOr(A.status, MHB_STATUS_BAD_PARAM);
            w = 1;
            c = 0;
        }
    } else {
        w = 1;
        c = 0;
    }
    LaneTab t;
    t.A = w;
    t.Ap = companion_fast(w, p);
    t.B = c;
    if (A.fpq) {  // float-quotient lanes (walk2_random_fpq): rd(w/p) and c + 2^23-magic * p
        t.Ap = __float_as_uint(__double2float_rd((double)w / (double)p));
        t.B = c + 0x4B000000u * p;
    }
    t.pad = 0;
    A.tab[i] = t;
    InvTab v;
    v.B = c;
    v.inv = inv_mod(w, p);
    v.invp = companion_fast(v.inv, p);
    // -c * w^{-1} mod p: the argmin is then one multiply-add, (h * w^{-1} + pad) mod p
    const uint32_t cw = reduce_once(shoup_lazy(v.inv, v.invp, c, p), p);
    v.pad = cw ? p - cw : 0u;
    A.inv[i] = v;
}

template <typename OutT>
__global__ void plan_count_kernel(SignArgs A) {
    __shared__ unsigned sh[kChunk];
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;

    for (int64_t i = tid; i < A.n_tot; i += stride) fill_lane_tables(A, i);

    for (int64_t s = tid; s < A.n_sets; s += stride) {
        const int64_t n = A.indptr[s + 1] - A.indptr[s];
        if (n <= 0) {
            if (A.status) atomicOr(A.status, MHB_STATUS_EMPTY_SET);
            continue;
        }
        const int64_t nch = (n + A.chunk - 1) / A.chunk;
        const int last = (int)(n - (nch - 1) * A.chunk);
        atomicAdd(&sh[last - 1], 1u);
        if (nch > 1) {
            atomicAdd(&sh[A.chunk - 1], (unsigned)(nch - 1));
            const unsigned long long k = atomicAdd(&A.sched->n_big, 1ull);
            A.big[k] = s;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x)
        if (sh[i]) atomicAdd(&A.hist[i], sh[i]);
}

// Rows A.big[e0 .. n_big) (strided by the grid's warps) start at UINT_MAX: one warp per
// row, the next row's index loaded while this one is written (a block per row with the
// index load on the critical path took 108 us for cfg2's 27k long sets at 256-id chunks).
template <typename OutT>
__device__ __forceinline__ void init_long_rows(const SignArgs& A, unsigned long long b0, unsigned long long nb,
                                               unsigned long long n_big) {
    const int lane = threadIdx.x & 31;
    const unsigned long long nw = blockDim.x >> 5;
    const unsigned long long stride = nb * nw;
    unsigned long long e = b0 * nw + (threadIdx.x >> 5);
    OutT* out = reinterpret_cast<OutT*>(A.out);
    int64_t s = e < n_big ? A.big[e] : 0;
    while (e < n_big) {
        const unsigned long long en = e + stride;
        const int64_t sn = en < n_big ? A.big[en] : 0;
        OutT* row = out + s * (int64_t)A.n_hash;
        for (int i = lane; i < A.n_hash; i += 32) row[i] = (OutT)(~0u);
        e = en;
        s = sn;
    }
}

// One block of kChunk threads: cursor[size-1] = number of virtual sets larger than
// `size` (descending order), total -> sched->n_vsets.
__global__ void plan_scan_kernel(SignArgs A) {
    __shared__ unsigned warp_tot[kChunk / 32];
    const int t = threadIdx.x;               // t-th largest size: size = kChunk - t
    const int bin = kChunk - 1 - t;
    const unsigned v = A.hist[bin];
    unsigned incl = v;
    const int lane = t & 31, w = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
        unsigned x = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        warp_tot[lane] = x;  // inclusive prefix of warp totals
    }
    __syncthreads();
    const unsigned base = w > 0 ? warp_tot[w - 1] : 0u;
    A.hist[kChunk + bin] = base + incl - v;  // exclusive start of this size's run
    if (t == kChunk - 1) A.sched->n_vsets = base + incl;
}

// Place every virtual set at its sorted position.  Each block owns a contiguous
// range of sets: it counts its virtual sets per size in shared memory, reserves
// one run per size with a single global atomic, then places them (hot size bins
// see one global atomic per block instead of one per set).  Afterwards the blocks
// initialise the output rows of long sets (merged with atomicMin) to UINT_MAX.
template <typename OutT>
__global__ void plan_scatter_kernel(SignArgs A) {
    __shared__ unsigned cnt[kChunk];
    __shared__ unsigned base[kChunk];
    unsigned* cursor = A.hist + kChunk;
    const int64_t per = (A.n_sets + gridDim.x - 1) / gridDim.x;
    const int64_t s_begin = (int64_t)blockIdx.x * per;
    const int64_t s_end = min(A.n_sets, s_begin + per);
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int64_t s = s_begin + threadIdx.x; s < s_end; s += blockDim.x) {
        const int64_t n = A.indptr[s + 1] - A.indptr[s];
        if (n <= 0) continue;
        const int64_t nch = (n + A.chunk - 1) / A.chunk;
        atomicAdd(&cnt[(int)(n - (nch - 1) * A.chunk) - 1], 1u);
        if (nch > 1) atomicAdd(&cnt[A.chunk - 1], (unsigned)(nch - 1));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x) {
        base[i] = cnt[i] ? atomicAdd(&cursor[i], cnt[i]) : 0u;
        cnt[i] = 0;
    }
    __syncthreads();
    for (int64_t s = s_begin + threadIdx.x; s < s_end; s += blockDim.x) {
        const int64_t lo = A.indptr[s];
        const int64_t n = A.indptr[s + 1] - lo;
        if (n <= 0) continue;
        const int64_t nch = (n + A.chunk - 1) / A.chunk;
        const long long merge = nch > 1 ? 1 : 0;
        // the nch - 1 full chunks take one run of the `chunk` bin with a single atomic
        // (one per chunk serialised on that bin: 108 us at 256-id chunks of cfg2)
        unsigned pos_full = 0;
        if (nch > 1) pos_full = base[A.chunk - 1] + atomicAdd(&cnt[A.chunk - 1], (unsigned)(nch - 1));
        for (int64_t c = 0; c + 1 < nch; ++c) {
            VSet v;
            v.f0 = lo + c * A.chunk;
            v.meta = ((long long)s << 12) | (merge << 11) | (long long)(A.chunk - 1);
            A.vsets[pos_full + c] = v;
        }
        const int size = (int)(n - (nch - 1) * A.chunk);
        VSet v;
        v.f0 = lo + (nch - 1) * A.chunk;
        v.meta = ((long long)s << 12) | (merge << 11) | (long long)(size - 1);
        A.vsets[base[size - 1] + atomicAdd(&cnt[size - 1], 1u)] = v;
    }
    // rows of long sets start at UINT_MAX (their chunks merge with atomicMin)
    const unsigned long long n_big = *((volatile unsigned long long*)&A.sched->n_big);
    init_long_rows<OutT>(A, blockIdx.x, gridDim.x, n_big);
}

// Small batches (n_sets <= kSmallPlan = 16384): the whole plan in ONE launch.  No size
// sort: virtual sets stay in set order (each set's chunks consecutive), placed by a
// single-pass prefix sum of the chunk counts over tiles of kSmallTile sets, one tile
// per CTA: every CTA publishes its tile's aggregate, then sums the aggregates of the
// tiles before it in parallel (a CTA takes its tile from a ticket counter and waits
// only for tiles whose tickets were taken before its own -- CTAs already running).  The three sorted-plan kernels
// cost ~16 us at 10,000 sets; a one-CTA plan ~24 us (one SM, latency-bound).  A warp
// group then holds sets of unequal sizes, so sign_small_batch_kernel runs the group's
// largest part (a warp max).  Lane tables: every CTA fills a slice.
constexpr int64_t kSmallPlan = kSmallPlanSets;
// The enumerating kernel (gap.cu) where its cost model prefers it.  Batches that the
// one-launch small-batch plan could take go to it only with a full wave of tiles (below
// that the small-batch kernel's finer work items fill the SMs better: cfg4 shapes cross
// over near 4,096 sets, cfg3 shapes near 12,000).
static bool gap_wanted(int kind, uint64_t prime, int32_t n_hash, int64_t n_sets, int64_t nnz) {
    if (!gap_preferred(kind, prime, n_hash, n_sets, nnz)) return false;
    if (n_sets > kSmallPlan) return true;
    const char* e = std::getenv("MHB_GAP_MIN_SETS");
    return n_sets >= (e ? std::atoll(e) : gap_full_wave_sets(n_hash, n_sets, nnz));
}
constexpr int kSmallTile = 256;  // sets per tile = threads per CTA

// hist[] doubles as the look-back state: [0] ticket counter, [2 + 2k] / [3 + 2k] tile
// k's (chunks, long sets) aggregate + 1 (0 = not yet published).
template <typename OutT>
__device__ __forceinline__ void plan_small_tile(const SignArgs& A, unsigned tile, unsigned n_tiles, unsigned* warp_c,
                                                unsigned* warp_b, unsigned& excl_c, unsigned& excl_b,
                                                unsigned* warp_tot2, unsigned* warp_totb2) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    volatile unsigned* flags = A.hist;
    const int64_t s = (int64_t)tile * kSmallTile + t;
    int64_t lo = 0, n = 0;
    if (s < A.n_sets) {
        lo = A.indptr[s];
        n = A.indptr[s + 1] - lo;
    }
    unsigned chunks = 0, bigs = 0;
    if (s < A.n_sets) {
        if (n <= 0) {
            if (A.status) atomicOr(A.status, MHB_STATUS_EMPTY_SET);
        } else {
            const int64_t nch = (n + A.chunk - 1) / A.chunk;
            chunks = (unsigned)nch;
            bigs = nch > 1 ? 1u : 0u;
        }
    }
    unsigned ci = chunks, bi = bigs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, ci, o), z = __shfl_up_sync(0xffffffffu, bi, o);
        if (lane >= o) {
            ci += y;
            bi += z;
        }
    }
    if (lane == 31) {
        warp_c[w] = ci;
        warp_b[w] = bi;
    }
    __syncthreads();
    if (t == 0) {
        unsigned tc = 0, tb = 0;
        for (int k = 0; k < kSmallTile / 32; ++k) {
            const unsigned c = warp_c[k], b = warp_b[k];
            warp_c[k] = tc;
            warp_b[k] = tb;
            tc += c;
            tb += b;
        }
        // publish this tile's aggregate at once (no waiting): every tile's prefix is
        // the sum of the aggregates before it, read in parallel below
        flags[3 + 2 * tile] = tb + 1u;
        __threadfence();
        flags[2 + 2 * tile] = tc + 1u;
        excl_c = tc;  // own aggregate, for the last tile's totals
        excl_b = tb;
    }
    __syncthreads();
    const unsigned own_c = excl_c, own_b = excl_b;
    // exclusive prefix = sum over tiles < tile of their aggregates (<= 64 tiles: two warps)
    if (w < 2) {
        unsigned pc = 0, pb = 0;
        const unsigned k = (unsigned)t;
        if (k < tile) {
            unsigned fc, fb;
            do {
                fc = flags[2 + 2 * k];
                fb = flags[3 + 2 * k];
            } while (fc == 0u || fb == 0u);
            pc = fc - 1u;
            pb = fb - 1u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pc += __shfl_xor_sync(0xffffffffu, pc, o);
            pb += __shfl_xor_sync(0xffffffffu, pb, o);
        }
        if (lane == 0) {
            warp_tot2[w] = pc;
            warp_totb2[w] = pb;
        }
    }
    __syncthreads();
    if (t == 0) {
        const unsigned pc = warp_tot2[0] + warp_tot2[1], pb = warp_totb2[0] + warp_totb2[1];
        excl_c = pc;
        excl_b = pb;
        if (tile + 1 == n_tiles) {
            A.sched->next = 0;
            A.sched->n_vsets = pc + own_c;
            A.sched->n_big = pb + own_b;
        }
    }
    __syncthreads();
    if (chunks) {
        unsigned pos = excl_c + warp_c[w] + ci - chunks;
        const long long merge = chunks > 1 ? 1 : 0;
        for (unsigned c = 0; c < chunks; ++c) {
            const int size = (int)((c + 1 < chunks) ? A.chunk : n - (int64_t)c * A.chunk);
            VSet vs;
            vs.f0 = lo + (int64_t)c * A.chunk;
            vs.meta = ((long long)s << 12) | (merge << 11) | (long long)(size - 1);
            A.vsets[pos++] = vs;
        }
        if (merge) A.big[excl_b + warp_b[w] + bi - bigs] = s;
    }
    // rows of this tile's long sets start at UINT_MAX (their chunks merge with
    // red.global.min): the CTA's warps share them
    if (own_b) {
        __syncthreads();
        const int lane = t & 31;
        for (unsigned e = excl_b + w; e < excl_b + own_b; e += kSmallTile / 32) {
            OutT* row = reinterpret_cast<OutT*>(A.out) + A.big[e] * (int64_t)A.n_hash;
            for (int i = lane; i < A.n_hash; i += 32) row[i] = (OutT)(~0u);
        }
    }
}

template <typename OutT>
__global__ void __launch_bounds__(kSmallTile) plan_small_kernel(SignArgs A, int32_t* status_out) {
    __shared__ unsigned warp_c[kSmallTile / 32], warp_b[kSmallTile / 32];
    __shared__ unsigned tile_s, excl_c, excl_b, warp_tot2[2], warp_totb2[2];
    const int t = threadIdx.x;
    // the caller's status word: zeroed here, ORed by sign_small_batch_kernel (which also
    // adds the flags this plan raises in the workspace word)
    if (blockIdx.x == 0 && t == 0 && status_out) *status_out = 0;
    if (t == 0) tile_s = atomicAdd(&A.hist[0], 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const unsigned n_tiles = (unsigned)((A.n_sets + kSmallTile - 1) / kSmallTile);
    // the first n_tiles tickets take the set tiles, the rest the lane tables: the two
    // latency chains (tile look-back; the lanes' modular inverses) run side by side
    if (tile < n_tiles) {
        plan_small_tile<OutT>(A, tile, n_tiles, warp_c, warp_b, excl_c, excl_b, warp_tot2, warp_totb2);
    } else {
        const unsigned n_lane_ctas = gridDim.x - n_tiles;
        for (int64_t i = (int64_t)(tile - n_tiles) * kSmallTile + t; i < A.n_tot;
             i += (int64_t)n_lane_ctas * kSmallTile)
            fill_lane_tables(A, i);
    }
}

// ----------------------------------------------------------------------------
// Walks
// ----------------------------------------------------------------------------

// Argmin recovery: x = (h - B_i) * A_i^{-1} mod p.
__device__ __forceinline__ uint32_t invert_entry(const InvTab& v, uint32_t h, uint32_t p) {
    uint32_t d = h - v.B;
    d = __viaddmin_u32(d, p, d);  // d in [0,p)
    return reduce_once(shoup_lazy(v.inv, v.invp, d, p), p);
}
// The same for 3p < 2^32 with one ALU instruction: x = h * A^{-1} + (-B A^{-1}) mod p
// (InvTab::pad), r = Shoup(h) + pad in [0, 3p); the two subtractions are IMADs by an
// opaque 1 (FMA pipe) and one VIMNMX3 picks the residue, as in start_hash_fma.
__device__ __forceinline__ uint32_t invert_entry_fma(const InvTab& v, uint32_t h, uint32_t negp, uint32_t one) {
    const uint32_t q = __umulhi(v.invp, h);
    const uint32_t r = v.inv * h + v.pad + q * negp;
    return __vimin3_u32(r, r * one + negp, r * one + 2u * negp);
}

// Long-set chunks merge with a fire-and-forget `red.global.min`.  Written as PTX:
// the C++ atomicMin in this loop makes ptxas move p out of the uniform datapath
// (every VIADDMNMX then reads -p from a vector register: -10% visit rate).
__device__ __forceinline__ void atomic_min_out(uint32_t* p, uint32_t v) {
    asm volatile("red.global.min.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void atomic_min_out(long long* p, uint32_t v) {
    asm volatile("red.global.min.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
}

__device__ __forceinline__ void store4(uint32_t* dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(a, b, c, d);
}
__device__ __forceinline__ void store4(long long* dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    longlong2* v = reinterpret_cast<longlong2*>(dst);
    v[0] = make_longlong2((long long)a, (long long)b);
    v[1] = make_longlong2((long long)c, (long long)d);
}

// Iterative walk over K lanes for two features at once.  Lookahead: h_{k+1} and
// h_{k+2} are both derived from h_k (steps dh and 2dh mod p), which halves the
// dependent chain and keeps the ALU pipe (VIADDMNMX + VIMNMX3) saturated
// (tools/visit_probe.cu: 41.9 visits/clk/SM vs 36.3 for the plain chain).
// FIRST: the group's first round initialises best instead of folding into it.
template <int K, bool FIRST>
__device__ __forceinline__ void walk2_iter(uint32_t (&best)[K], uint32_t ha, uint32_t da,
                                           uint32_t hb, uint32_t db, uint32_t p) {
    const uint32_t da2 = reduce_once(da + da, p), db2 = reduce_once(db + db, p);
#pragma unroll
    for (int k = 0; k < K; k += 2) {
        const uint32_t ga = reduce_once(ha + da, p), gb = reduce_once(hb + db, p);
        if (FIRST) {
            best[k] = min(ha, hb);
            best[k + 1] = min(ga, gb);
        } else {
            best[k] = __vimin3_u32(best[k], ha, hb);
            best[k + 1] = __vimin3_u32(best[k + 1], ga, gb);
        }
        if (k + 2 < K) {
            ha = reduce_once(ha + da2, p);
            hb = reduce_once(hb + db2, p);
        }
    }
}

template <int K>
__device__ __forceinline__ void walk1_iter(uint32_t (&best)[K], uint32_t ha, uint32_t da, uint32_t p) {
    const uint32_t da2 = reduce_once(da + da, p);
#pragma unroll
    for (int k = 0; k < K; k += 2) {
        best[k] = min(best[k], ha);
        best[k + 1] = min(best[k + 1], reduce_once(ha + da, p));
        if (k + 2 < K) ha = reduce_once(ha + da2, p);
    }
}

template <int K, bool NARROW, bool FIRST>
__device__ __forceinline__ void walk2_random(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                             const uint32_t (&cAp)[K], const uint32_t (&cB)[K],
                                             uint32_t xa, uint32_t xb, uint32_t p, uint32_t negp) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        uint32_t ra, rb;
        if (NARROW) {
            ra = mul_add_mod_narrow_n(cA[k], cAp[k], cB[k], xa, p, negp);
            rb = mul_add_mod_narrow_n(cA[k], cAp[k], cB[k], xb, p, negp);
        } else {
            ra = mul_add_mod_n(cA[k], cAp[k], cB[k], xa, p, negp);
            rb = mul_add_mod_n(cA[k], cAp[k], cB[k], xb, p, negp);
        }
        best[k] = FIRST ? min(ra, rb) : __vimin3_u32(best[k], ra, rb);
    }
}

template <int K, bool NARROW>
__device__ __forceinline__ void walk1_random(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                             const uint32_t (&cAp)[K], const uint32_t (&cB)[K],
                                             uint32_t xa, uint32_t p, uint32_t negp) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        uint32_t ra = NARROW ? mul_add_mod_narrow_n(cA[k], cAp[k], cB[k], xa, p, negp)
                             : mul_add_mod_n(cA[k], cAp[k], cB[k], xa, p, negp);
        best[k] = min(best[k], ra);
    }
}

// Random family, p <= 2^23: the Shoup quotient (IMAD.HI, two FMA-heavy issue slots)
// comes from the FP32 pipe instead.  With x < 2^23 exact in float and wf = rd(w/p),
// q = rz(x*wf + 2^23) - 2^23 = floor(x*wf) lies in {floor(x*w/p) - 1, floor(x*w/p)},
// so r = w*x + c - q*p lies in [0, 3p): two conditional subtracts.  The magic 2^23 is
// folded into the lane offset (cC = c + 0x4B000000 * p), q*p is added as bits*(2^32-p).
template <int K, bool FIRST>
__device__ __forceinline__ void walk2_random_fpq(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                                 const uint32_t (&cW)[K], const uint32_t (&cC)[K],
                                                 uint32_t xa, uint32_t xb, uint32_t p, uint32_t negp) {
    const float fa = __uint2float_rn(xa), fb = __uint2float_rn(xb);  // exact: x < 2^24
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float wf = __uint_as_float(cW[k]);
        const uint32_t qa = __float_as_uint(__fmaf_rz(fa, wf, 8388608.0f));
        const uint32_t qb = __float_as_uint(__fmaf_rz(fb, wf, 8388608.0f));
        const uint32_t ra = reduce_once(reduce_once(cA[k] * xa + cC[k] + qa * negp, p), p);
        const uint32_t rb = reduce_once(reduce_once(cA[k] * xb + cC[k] + qb * negp, p), p);
        best[k] = FIRST ? min(ra, rb) : __vimin3_u32(best[k], ra, rb);
    }
}

template <int K>
__device__ __forceinline__ void walk1_random_fpq(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                                 const uint32_t (&cW)[K], const uint32_t (&cC)[K], uint32_t xa,
                                                 uint32_t p, uint32_t negp) {
    const float fa = __uint2float_rn(xa);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t qa = __float_as_uint(__fmaf_rz(fa, __uint_as_float(cW[k]), 8388608.0f));
        best[k] = min(best[k], reduce_once(reduce_once(cA[k] * xa + cC[k] + qa * negp, p), p));
    }
}

// Per-thread hashing state: iterative start constants, or the K random-family lane constants.
template <int K, bool ITER>
struct LaneState {
    uint32_t tA, tAp, tB;
    uint32_t negp;  // 2^32 - p (kernel parameter)
    uint32_t one;   // opaque 1 (kernel parameter), see Spelling
    uint32_t cA[ITER ? 1 : K], cAp[ITER ? 1 : K], cB[ITER ? 1 : K];
};

// Per-instantiation spelling of the main loop.  The options are semantically identical;
// they steer ptxas's register assignment, whose register-bank conflicts move the visit
// rate by several percent.  Chosen per kernel with
// tools/variant_search.py (static bank-conflict score of the loop) and confirmed with
// tools/ab.sh on the B200; every other instantiation keeps the plain spelling.
#ifndef MHB_BV_START
#define MHB_BV_START 1
#endif
#ifndef MHB_BV_MAXID
#define MHB_BV_MAXID 1
#endif
#ifndef MHB_BV_SWAP
#define MHB_BV_SWAP 1
#endif
#ifndef MHB_BV_ADDR
#define MHB_BV_ADDR 1
#endif
#ifndef MHB_BV_U1
#define MHB_BV_U1 0
#endif
#ifndef MHB_BV_NREG
#define MHB_BV_NREG 120
#endif
#ifndef MHB_SV_ADDR
#define MHB_SV_ADDR 0
#endif
#ifndef MHB_SV_NREG
#define MHB_SV_NREG 120  // staged loop + prefetching fallback: 120 (bank score 72) 31.00 ms; 116 (100); 108 (38) 32.0
#endif
#ifndef MHB_SV_START
#define MHB_SV_START 1
#endif
#ifndef MHB_RV_NREG
#define MHB_RV_NREG 112
#endif
#ifndef MHB_RV_ADDR
#define MHB_RV_ADDR 1
#endif
#ifndef MHB_HV_NREG
#define MHB_HV_NREG 128
#endif
#ifndef MHB_HV_ADDR
#define MHB_HV_ADDR 0
#endif
#ifndef MHB_IV_NREG
#define MHB_IV_NREG 120
#endif
#ifndef MHB_IV_ADDR
#define MHB_IV_ADDR 1
#endif
#ifndef MHB_IV_START
#define MHB_IV_START 1
#endif
#ifndef MHB_SV_MAXID
#define MHB_SV_MAXID 1
#endif
#ifndef MHB_SV_SWAP
#define MHB_SV_SWAP 0
#endif
#ifndef MHB_RV_STAGE
#define MHB_RV_STAGE 1  // float-quotient random kernel (cfg3: one set per warp): 12.88 -> 12.36 ms at 112 registers
#endif
#ifndef MHB_BV_STAGE
#define MHB_BV_STAGE 0  // fused band keys staged like the cfg4 kernel: best of 20 spellings 31.95 ms vs 31.82
#endif
#ifndef MHB_SV_INVF
#define MHB_SV_INVF 0  // cfg4: 31.01 -> 31.37 ms (register assignment); cfg2/cfg3 kernel +0.45%
#endif
#ifndef MHB_IV_INVF
#define MHB_IV_INVF 1  // cfg2 4.698 -> 4.676 ms, cfg3 5.672 -> 5.648 ms (A/B, 3 rounds)
#endif
#ifndef MHB_RV_INVF
#define MHB_RV_INVF 0  // float-quotient kernel: loop bank score 52 -> 80
#endif
#ifndef MHB_SV_STAGE
#define MHB_SV_STAGE 1  // cfg4 kernel: ids staged per set (see Spelling::staged)
#endif
template <int K, bool ITER, bool NARROW, bool FPQ, bool SKEW, bool BANDS>
struct Spelling {
    static constexpr bool kIter64 = ITER && NARROW && K == 64 && (!BANDS || SKEW);  // cfg1-5 iterative kernels
    static constexpr bool kBands64 = kIter64 && BANDS;  // cfg4 fused band keys (MHB_BV_*: A/B knobs)
    static constexpr bool kSkew64 = kIter64 && SKEW && !BANDS;  // cfg4 signatures only (MHB_SV_*)
    static constexpr bool kFpq = FPQ && !BANDS;                 // cfg1/cfg3 random family (MHB_RV_*)
    static constexpr bool kPlain64 = kIter64 && !SKEW && !BANDS;  // cfg1/2/3/5 iterative (MHB_IV_*)
    static constexpr bool kShoup = !ITER && !FPQ && !BANDS;        // random family, p > 2^23 (MHB_HV_*)
    // start hash: min(r, r - p, r - 2p) with both subtractions as IMADs by an opaque 1
    // (FMA pipe; plain subtractions fold into two VIADDMNMX on the ALU pipe)
    static constexpr bool start_fma = kBands64 ? MHB_BV_START : kSkew64 ? MHB_SV_START : kPlain64 ? MHB_IV_START : kIter64;
    // round loop: the id maximum after the round, the features passed as (b, a)
    static constexpr bool maxid_after = kBands64 ? MHB_BV_MAXID : kSkew64 ? MHB_SV_MAXID : kIter64;
    static constexpr bool swap_features = kBands64 ? MHB_BV_SWAP : kSkew64 ? MHB_SV_SWAP : kIter64;
    // id address as one IMAD.WIDE by an opaque 4 instead of IADD3 + LEA + LEA.HI.X
    static constexpr bool addr_fma = kBands64 ? MHB_BV_ADDR : kSkew64 ? MHB_SV_ADDR : kFpq ? MHB_RV_ADDR
                                    : kPlain64 ? MHB_IV_ADDR : kShoup ? MHB_HV_ADDR : false;
    static constexpr int maxnreg = kBands64 ? MHB_BV_NREG : kSkew64 ? MHB_SV_NREG : kFpq ? MHB_RV_NREG
                                   : kPlain64 ? MHB_IV_NREG : kShoup ? MHB_HV_NREG : 128;
    // one set per warp (F == 1, N >= 2048): the set's ids staged in shared memory and
    // walked with LDS.64 pairs -- no address arithmetic or clamps in the round loop
    // invalid slots' size / first id read without a valid check (load_vset): cfg2/cfg3
    // iterative +1.1%, the Shoup random kernel -5% (its bank-conflict score 51 -> 59)
    static constexpr bool plain_meta = kIter64 && !BANDS;  // (the band-key loop: score 72 -> 107)
    // argmin recovery in the epilogue fast path with one ALU instruction per entry
    static constexpr bool inv_fma = NARROW && !BANDS && (kSkew64 ? MHB_SV_INVF : kPlain64 ? MHB_IV_INVF : kFpq ? MHB_RV_INVF : false);
    static constexpr bool staged = (kSkew64 && MHB_SV_STAGE) || (kBands64 && SKEW && MHB_BV_STAGE) || (kFpq && MHB_RV_STAGE);
};
// u32 per staging buffer of the staged kernels (sets of <= 241 ids; two buffers per warp keep two
// 256-thread CTAs of the cfg4 kernel on an SM: 64 KB dump rows + 33 KB epilogue table + 15.6 KB)
constexpr int kSetStage = 244;

// Start hash h_{i0}(x) for 3p < 2^32 (see Spelling::start_fma).
template <int K, bool ITER>
__device__ __forceinline__ uint32_t start_hash_fma(const LaneState<K, ITER>& ls, uint32_t x) {
    const uint32_t q = __umulhi(ls.tAp, x);
    const uint32_t r = ls.tA * x + ls.tB + q * ls.negp;
    return __vimin3_u32(r, r * ls.one + ls.negp, r * ls.one + 2u * ls.negp);
}

// ids[base + j] (see Spelling::addr_fma).
__device__ __forceinline__ uint32_t ld_id_fma(const uint32_t* base, uint32_t j, uint32_t four) {
    const uint32_t* a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(j), "r"(four), "l"(base));
    return __ldg(a);
}

template <int K, bool ITER, bool NARROW, bool FIRST, bool FPQ = false, bool START_FMA = false>
__device__ __forceinline__ void round2(uint32_t (&best)[K], const LaneState<K, ITER>& ls, uint32_t xa, uint32_t xb,
                                       uint32_t p, uint32_t bpar) {
    if constexpr (ITER) {
        // NARROW (3p < 2^32): the start hashes reduce with one VIMNMX3 each
        const uint32_t ha = START_FMA ? start_hash_fma(ls, xa)
                            : NARROW  ? mul_add_mod_min3(ls.tA, ls.tAp, ls.tB, xa, p)
                                      : mul_add_mod(ls.tA, ls.tAp, ls.tB, xa, p);
        const uint32_t hb = START_FMA ? start_hash_fma(ls, xb)
                            : NARROW  ? mul_add_mod_min3(ls.tA, ls.tAp, ls.tB, xb, p)
                                      : mul_add_mod(ls.tA, ls.tAp, ls.tB, xb, p);
        walk2_iter<K, FIRST>(best, ha, reduce_once(xa + bpar, p), hb, reduce_once(xb + bpar, p), p);
    } else if constexpr (FPQ) {
        walk2_random_fpq<K, FIRST>(best, ls.cA, ls.cAp, ls.cB, xa, xb, p, ls.negp);
    } else {
        walk2_random<K, NARROW, FIRST>(best, ls.cA, ls.cAp, ls.cB, xa, xb, p, ls.negp);
    }
}

template <int K, bool ITER, bool NARROW, bool FPQ = false, bool START_FMA = false>
__device__ __forceinline__ void round1(uint32_t (&best)[K], const LaneState<K, ITER>& ls, uint32_t xa,
                                       uint32_t p, uint32_t bpar) {
    if constexpr (ITER) {
        const uint32_t ha = START_FMA ? start_hash_fma(ls, xa)
                            : NARROW  ? mul_add_mod_min3(ls.tA, ls.tAp, ls.tB, xa, p)
                                      : mul_add_mod(ls.tA, ls.tAp, ls.tB, xa, p);
        walk1_iter<K>(best, ha, reduce_once(xa + bpar, p), p);
    } else if constexpr (FPQ) {
        walk1_random_fpq<K>(best, ls.cA, ls.cAp, ls.cB, xa, p, ls.negp);
    } else {
        walk1_random<K, NARROW>(best, ls.cA, ls.cAp, ls.cB, xa, p, ls.negp);
    }
}

// ----------------------------------------------------------------------------
// Main kernel
// ----------------------------------------------------------------------------

// The slice's virtual set for work item `it` (group = it / n_super), or an
// invalid entry past the end: f0 = 0 and meta = -4096 (negative, size field 0), so a
// slot's size and first id read the same way whether it is valid or not.
__device__ __forceinline__ VSet load_vset(const SignArgs& A, unsigned long long it, unsigned long long n_vsets,
                                          int f) {
    VSet v;
    v.f0 = 0;
    v.meta = -4096;
    const unsigned long long group = A.n_super == 1 ? it : it / (unsigned)A.n_super;
    const unsigned long long k = (group << A.log2F) + f;
    if (k < n_vsets) v = A.vsets[k];
    return v;
}

// Dump a thread's K minima into its (swizzled) smem row, then invert and store them
// four lanes at a time.  EPI_SMEM: epilogue table staged in shared memory.
template <int K>
__device__ __forceinline__ void dump_best(const uint32_t (&best)[K], uint32_t* row, int lane) {
    constexpr int NQ = K / 4;
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
        *reinterpret_cast<uint4*>(row + ((q ^ (lane & SWZ)) << 2)) =
            make_uint4(best[4 * q], best[4 * q + 1], best[4 * q + 2], best[4 * q + 3]);
}

template <int K>
__host__ __device__ constexpr int kLog2() { return K <= 1 ? 0 : 1 + kLog2<K / 2>(); }

// SKEW: the shared-memory epilogue table holds lane i at i + i/K.  With large G (lane
// blocks of the warp's threads K apart, N >= 16*K) the 8 threads of an LDS.128 phase
// would otherwise all hit one bank group (an 8-way conflict at G = 32).
template <int K, typename OutT, bool EPI_SMEM, bool BANDS, bool SKEW, bool UNROLL, bool INV_FMA = false>
__device__ __forceinline__ void emit_lanes(const SignArgs& A, const uint32_t* dump_row, int lane, int64_t set,
                                           bool merge, int64_t i0, const InvTab* epi_s, uint32_t negp = 0,
                                           uint32_t one = 1) {
    constexpr int NQ = K / 4;
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;
    const uint32_t p = A.p;
    const int32_t N = A.n_hash;
    const bool vec_ok = (N & 3) == 0;
    OutT* row = reinterpret_cast<OutT*>(A.out) + set * (int64_t)N;
    if constexpr (EPI_SMEM && !BANDS) {
        // Common case: the thread's whole lane block lies inside the row.  i0 is a
        // multiple of K, so the skew is one offset for the block and every index is a
        // 32-bit constant offset: no per-quad bounds or 64-bit index arithmetic.
        const int j0 = (int)i0;
        if (!merge && vec_ok && j0 + K <= N) {
            const InvTab* t = epi_s + (SKEW ? j0 + j0 / K : j0);
            OutT* r = row + j0;
            // UNROLL (skewed and float-quotient kernels): +0.8..3%; the cfg2/cfg3 iterative
            // and Shoup random kernels lose 0.4..1% to the register assignment it brings
#pragma unroll(UNROLL ? 4 : 1)
            for (int q = 0; q < NQ; ++q) {
                const uint4 m = *reinterpret_cast<const uint4*>(dump_row + ((q ^ (lane & SWZ)) << 2));
                if constexpr (INV_FMA)
                    store4(r + 4 * q, invert_entry_fma(t[4 * q], m.x, negp, one),
                           invert_entry_fma(t[4 * q + 1], m.y, negp, one), invert_entry_fma(t[4 * q + 2], m.z, negp, one),
                           invert_entry_fma(t[4 * q + 3], m.w, negp, one));
                else
                    store4(r + 4 * q, invert_entry(t[4 * q], m.x, p), invert_entry(t[4 * q + 1], m.y, p),
                           invert_entry(t[4 * q + 2], m.z, p), invert_entry(t[4 * q + 3], m.w, p));
            }
            return;
        }
    }
    if constexpr (EPI_SMEM && BANDS) {
        // The same fast path with the band keys hashed as the argmins come out: a band is
        // rows/4 whole quads of this thread's block (rows divides K), so a quad countdown
        // replaces the per-quad band arithmetic of the general loop below.
        const int j0 = (int)i0;
        if (!merge && vec_ok && j0 + K <= N) {
            const InvTab* t = epi_s + (SKEW ? j0 + j0 / K : j0);
            OutT* r = row + j0;
            const int rq = A.rows >> 2;  // quads per band
            unsigned long long* key = A.keys + set * (int64_t)(N / A.rows) + j0 / A.rows;
            BandHash hk(0u);
            int left = 0;
#pragma unroll(UNROLL ? 4 : 1)
            for (int q = 0; q < NQ; ++q) {
                const uint4 m = *reinterpret_cast<const uint4*>(dump_row + ((q ^ (lane & SWZ)) << 2));
                const uint32_t x0 = invert_entry(t[4 * q], m.x, p), x1 = invert_entry(t[4 * q + 1], m.y, p);
                const uint32_t x2 = invert_entry(t[4 * q + 2], m.z, p), x3 = invert_entry(t[4 * q + 3], m.w, p);
                if (left == 0) {
                    hk = BandHash((uint32_t)((j0 + 4 * q) / A.rows));
                    left = rq;
                }
                hk.add(x0);
                hk.add(x1);
                hk.add(x2);
                hk.add(x3);
                if (--left == 0) *key++ = hk.key();
                if (A.write_sig) store4(r + 4 * q, x0, x1, x2, x3);
            }
            return;
        }
    }
    BandHash hk(0u);  // running band hash (BANDS)
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
        const int64_t i = i0 + 4 * q;
        if (i >= N) break;
        const uint4 m = *reinterpret_cast<const uint4*>(dump_row + ((q ^ (lane & SWZ)) << 2));
        const uint32_t h[4] = {m.x, m.y, m.z, m.w};
        if (merge) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (i + e < N) atomic_min_out(row + i + e, h[e]);
            continue;
        }
        uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t ie = SKEW ? (i + e) + ((i + e) >> kLog2<K>()) : i + e;
            const InvTab t = EPI_SMEM ? epi_s[ie] : A.inv[min(i + e, A.n_tot - 1)];
            x[e] = invert_entry(t, h[e], p);
        }
        if constexpr (BANDS) {
            // bands are runs of A.rows lanes; rows divides K and n_hash, so a band never
            // straddles threads or the row end
            const int64_t band = i / A.rows;
            if (i - band * A.rows == 0) hk = BandHash((uint32_t)band);
#pragma unroll
            for (int e = 0; e < 4; ++e) hk.add(x[e]);
            if (i + 4 - band * A.rows == A.rows) A.keys[set * (int64_t)(N / A.rows) + band] = hk.key();
            if (!A.write_sig) continue;
        }
        if (vec_ok && i + 3 < N) {
            store4(row + i, x[0], x[1], x[2], x[3]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (i + e < N) row[i + e] = (OutT)x[e];
        }
    }
}

// Long sets: rows hold min hash values after the main kernel; invert in place
// (one block per row, threads over hash lanes).
__device__ __forceinline__ void cpa4(uint32_t saddr, const uint32_t* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}

template <typename OutT>
__device__ __forceinline__ void finalize_rows(const SignArgs& A, unsigned long long e0, unsigned long long stride) {
    // one warp per row (block e0 of `stride` blocks), the next row's index loaded ahead
    const unsigned long long n_big = *((volatile unsigned long long*)&A.sched->n_big);
    OutT* out = reinterpret_cast<OutT*>(A.out);
    const int lane = threadIdx.x & 31;
    const unsigned long long nw = blockDim.x >> 5;
    const unsigned long long step = stride * nw;
    unsigned long long e = e0 * nw + (threadIdx.x >> 5);
    int64_t s = e < n_big ? A.big[e] : 0;
    while (e < n_big) {
        const unsigned long long en = e + step;
        const int64_t sn = en < n_big ? A.big[en] : 0;
        OutT* row = out + s * (int64_t)A.n_hash;
#pragma unroll 4
        for (int i = lane; i < A.n_hash; i += 32) row[i] = (OutT)invert_entry(A.inv[i], (uint32_t)row[i], A.p);
        if (A.keys) {  // band keys of long sets (their chunks merged in `out`)
            __syncwarp();
            const int n_bands = A.n_hash / A.rows;
            for (int band = lane; band < n_bands; band += 32) {
                BandHash hk((uint32_t)band);
                for (int j = 0; j < A.rows; ++j) hk.add((uint32_t)row[band * A.rows + j]);
                A.keys[s * (int64_t)n_bands + band] = hk.key();
            }
            __syncwarp();
        }
        e = en;
        s = sn;
    }
}

// p and b arrive as separate scalar parameters so ptxas keeps them in uniform
// registers: VIADDMNMX t, -UR, t reads one vector register instead of two
// (tools/visit_probe.cu: 41.9 vs 37.8 visits/clk/SM).
template <int K, bool ITER, bool NARROW, typename OutT, bool BANDS = false, bool FPQ = false, bool SKEW = false>
__global__ void __maxnreg__((Spelling<K, ITER, NARROW, FPQ, SKEW, BANDS>::maxnreg))  // 128: 2 CTAs of 256 per SM
sign_kernel(SignArgs A, uint32_t p, uint32_t bpar, uint32_t negp, uint32_t one) {
    using S = Spelling<K, ITER, NARROW, FPQ, SKEW, BANDS>;
    extern __shared__ uint4 smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* dump_row = reinterpret_cast<uint32_t*>(smem_raw) + (warp * 32 + lane) * K;
    InvTab* epi_s = reinterpret_cast<InvTab*>(reinterpret_cast<uint32_t*>(smem_raw) + kBlock * K);

    const int F = A.F;
    const int g = lane >> A.log2F;
    const int f = lane & (F - 1);

    // Stage the epilogue table (B_i, A_i^{-1}, companion) in shared memory.
    const bool epi_smem = A.n_tot <= kEpiSmemLanes;
    if (epi_smem) {
        for (int i = threadIdx.x; i < A.n_tot; i += blockDim.x) epi_s[SKEW ? i + i / K : i] = A.inv[i];
        __syncthreads();
    }

    const unsigned long long n_vsets = *((volatile unsigned long long*)&A.sched->n_vsets);
    const unsigned long long n_groups = (n_vsets + F - 1) >> A.log2F;
    const unsigned long long n_items = n_groups * (unsigned)A.n_super;

    // Work items flow through a 3-deep pipeline: the id of the item after next is
    // claimed while the current one runs, the next item's set entry is loaded, and
    // the last round of the current item prefetches the next item's first features.
    // Items come from the counter (dynamic balance of the size-sorted work).
    unsigned long long it = 0, itn = 0, itnn = 0;
    if (lane == 0) {
        it = atomicAdd(&A.sched->next, 1ull);
        itn = atomicAdd(&A.sched->next, 1ull);
    }
    it = __shfl_sync(0xffffffffu, it, 0);
    itn = __shfl_sync(0xffffffffu, itn, 0);
    VSet ec = load_vset(A, it, n_vsets, f);
    VSet en = load_vset(A, itn, n_vsets, f);

    LaneState<K, ITER> ls;
    ls.negp = negp;
    ls.one = one;
    const uint32_t four = one << 2;
    int cur_sb = -1;
    uint32_t maxid = 0;

    if constexpr (S::staged) {
        if (F == 1) {
            // Every lane of the warp walks the same set.  Its ids (plus a copy of the last,
            // so an odd set's final pair is valid) are staged into one of two per-warp
            // buffers with cp.async while the previous item is walked; the rounds read
            // LDS.64 pairs.  Sets longer than the buffer walk from global memory.
            uint32_t* wbuf = reinterpret_cast<uint32_t*>(smem_raw) + kBlock * K +
                             (epi_smem ? 4 * (int)(A.n_tot + A.n_tot / K + 1) : 0) + warp * 2 * kSetStage;
            auto stage = [&](const VSet& v, int b) -> bool {
                const int n = v.meta >= 0 ? (int)(v.meta & 2047) + 1 : 0;
                const bool st = n > 0 && n + 3 <= kSetStage;
                if (st) {
                    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(wbuf + b * kSetStage);
                    const uint32_t* gsrc = A.ids + v.f0;
                    for (int j = lane; j <= n; j += 32) cpa4(sa + 4 * j, gsrc + min(j, n - 1));
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                return st;
            };
            int cur = 0;
            bool stc = stage(ec, 0);
            while (it < n_items) {
                if (lane == 0) itnn = atomicAdd(&A.sched->next, 1ull);
                const bool stn = stage(en, cur ^ 1);
                int sb = 0;
                if (A.n_super > 1) sb = (int)(it % (unsigned)A.n_super);
                if (sb != cur_sb) {
                    const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
                    if constexpr (ITER) {
                        const LaneTab t = A.tab[i0];
                        ls.tA = t.A; ls.tAp = t.Ap; ls.tB = t.B;
                    } else {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const LaneTab t = A.tab[i0 + k];
                            ls.cA[k] = t.A; ls.cAp[k] = t.Ap; ls.cB[k] = t.B;
                        }
                    }
                    cur_sb = sb;
                }
                const bool valid = ec.meta >= 0;
                const int n = __shfl_sync(0xffffffffu, valid ? (int)(ec.meta & 2047) + 1 : 1, 0);
                const int rounds = (n + 1) >> 1;
                uint32_t best[K];
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncwarp();
                if (stc) {
                    const uint32_t* b = wbuf + cur * kSetStage;
                    for (int j = lane; j < n; j += 32) maxid = max(maxid, b[j]);
                    uint2 v = *reinterpret_cast<const uint2*>(b);
                    uint2 nx = *reinterpret_cast<const uint2*>(b + 2);
                    round2<K, ITER, NARROW, true, FPQ, S::start_fma>(best, ls, v.x, v.y, p, bpar);
                    const uint2* pp = reinterpret_cast<const uint2*>(b + 4);
#pragma unroll 1
                    for (int r = 1; r < rounds; ++r) {
                        v = nx;
                        nx = *pp++;  // one pair ahead; past the set it reads unused buffer words
                        if constexpr (S::swap_features) round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, v.y, v.x, p, bpar);
                        else round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, v.x, v.y, p, bpar);
                    }
                } else {
                    // longer sets: global loads one round ahead (an odd set's last pair
                    // repeats its last id, harmless for a minimum)
                    const uint32_t* gsrc = A.ids + (valid ? ec.f0 : 0);
                    const int last = n - 1;
                    uint32_t xa = __ldg(gsrc), xb = __ldg(gsrc + min(1, last));
                    uint32_t na = __ldg(gsrc + min(2, last)), nb = __ldg(gsrc + min(3, last));
                    maxid = __vimax3_u32(maxid, xa, xb);
                    round2<K, ITER, NARROW, true, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
#pragma unroll 1
                    for (int r = 1; r < rounds; ++r) {
                        xa = na;
                        xb = nb;
                        na = __ldg(gsrc + min(2 * r + 2, last));
                        nb = __ldg(gsrc + min(2 * r + 3, last));
                        maxid = __vimax3_u32(maxid, xa, xb);
                        round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
                    }
                }
                if (valid) {
                    const int64_t set = ec.meta >> 12;
                    const bool merge = (ec.meta >> 11) & 1;
                    const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
                    dump_best<K>(best, dump_row, lane);
                    if (epi_smem) emit_lanes<K, OutT, true, BANDS, SKEW, true, S::inv_fma>(A, dump_row, lane, set, merge, i0, epi_s, negp, one);
                    else emit_lanes<K, OutT, false, BANDS, SKEW, true>(A, dump_row, lane, set, merge, i0, epi_s);
                }
                __syncwarp();  // the buffer is restaged two items later
                it = itn;
                ec = en;
                itn = __shfl_sync(0xffffffffu, itnn, 0);
                en = load_vset(A, itn, n_vsets, f);
                stc = stn;
                cur ^= 1;
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            if (__any_sync(0xffffffffu, maxid >= p) && lane == 0 && A.status) atomicOr(A.status, MHB_STATUS_ID_GE_PRIME);
            return;
        }
    }

    uint32_t xa = 0, xb = 0;
    {
        const int n = S::plain_meta || ec.meta >= 0 ? (int)(ec.meta & 2047) + 1 : 1;
        const uint32_t* base = A.ids + (S::plain_meta || ec.meta >= 0 ? ec.f0 : 0);
        xa = __ldg(base);
        xb = __ldg(base + min(1, n - 1));
    }

    while (it < n_items) {
        if (lane == 0) itnn = atomicAdd(&A.sched->next, 1ull);
        int sb = 0;
        if (A.n_super > 1) sb = (int)(it % (unsigned)A.n_super);
        if (sb != cur_sb) {  // lane constants change only with the lane pass
            const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
            if constexpr (ITER) {
                const LaneTab t = A.tab[i0];
                ls.tA = t.A; ls.tAp = t.Ap; ls.tB = t.B;
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const LaneTab t = A.tab[i0 + k];
                    ls.cA[k] = t.A; ls.cAp[k] = t.Ap; ls.cB[k] = t.B;
                }
            }
            cur_sb = sb;
        }

        const bool valid = ec.meta >= 0;
        // an invalid slot reads as one feature at ids[0] (load_vset); S::plain_meta drops
        // the valid checks ptxas otherwise rematerializes in the round loop
        const int n = S::plain_meta ? (int)(ec.meta & 2047) + 1 : valid ? (int)(ec.meta & 2047) + 1 : 1;
        const int last = n - 1;
        const uint32_t* base = A.ids + (S::plain_meta ? ec.f0 : valid ? ec.f0 : 0);
        // the group's first set is its largest (descending sort)
        const int n_max = __shfl_sync(0xffffffffu, n, 0);
        const int rounds = (n_max + 1) >> 1;
        const bool odd = n_max & 1;
        // next item's first features (cross-item prefetch)
        const bool nvalid = en.meta >= 0;
        const uint32_t* nbase = A.ids + (S::plain_meta ? en.f0 : nvalid ? en.f0 : 0);
        const int nlast = S::plain_meta ? (int)(en.meta & 2047) : nvalid ? (int)(en.meta & 2047) : 0;

        // Rounds of two features.  Ids are prefetched two rounds ahead inside the
        // item; the item's second-to-last round fetches the next item's first round.
        uint32_t best[K];
        if (rounds == 1) {
            const uint32_t pa = __ldg(nbase), pb = __ldg(nbase + min(1, nlast));
            maxid = __vimax3_u32(maxid, xa, xb);
            round2<K, ITER, NARROW, true, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
            xa = pa; xb = pb;
        } else {
            uint32_t pa = __ldg(base + min(2, last)), pb = __ldg(base + min(3, last));  // round 1
            uint32_t qa, qb;                                                    // round 2 / next item's 0
            if (rounds > 2) {
                qa = __ldg(base + min(4, last));
                qb = __ldg(base + min(5, last));
            } else {
                qa = __ldg(nbase);
                qb = __ldg(nbase + min(1, nlast));
            }
            maxid = __vimax3_u32(maxid, xa, xb);
            round2<K, ITER, NARROW, true, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
            xa = pa; xb = pb; pa = qa; pb = qb;
            int o = 6;
#pragma unroll 1
            for (int r = 1; r + 2 < rounds; ++r, o += 2) {
                // smaller sets of the group clamp to their last id
                if constexpr (S::addr_fma) {
                    qa = ld_id_fma(base, min(o, last), four);
                    qb = ld_id_fma(base, min(o + 1, last), four);
                } else {
                    qa = __ldg(base + min(o, last));
                    qb = __ldg(base + min(o + 1, last));
                }
                if constexpr (S::maxid_after) {
                    if constexpr (S::swap_features) round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xb, xa, p, bpar);
                    else round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
                    maxid = __vimax3_u32(maxid, xa, xb);
                } else {
                    maxid = __vimax3_u32(maxid, xa, xb);
                    round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
                }
                xa = pa; xb = pb; pa = qa; pb = qb;
            }
            if (rounds > 2) {
                qa = __ldg(nbase);
                qb = __ldg(nbase + min(1, nlast));
                maxid = __vimax3_u32(maxid, xa, xb);
                round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
                xa = pa; xb = pb; pa = qa; pb = qb;
            }
            if (odd) {
                maxid = max(maxid, xa);
                round1<K, ITER, NARROW, FPQ, S::start_fma>(best, ls, xa, p, bpar);
            } else {
                maxid = __vimax3_u32(maxid, xa, xb);
                round2<K, ITER, NARROW, false, FPQ, S::start_fma>(best, ls, xa, xb, p, bpar);
            }
            xa = pa; xb = pb;
        }

        if (valid) {
            const int64_t set = ec.meta >> 12;
            const bool merge = (ec.meta >> 11) & 1;
            const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
            dump_best<K>(best, dump_row, lane);
            if (epi_smem) emit_lanes<K, OutT, true, BANDS, SKEW, (SKEW && !(BANDS && MHB_BV_U1)) || FPQ, S::inv_fma>(A, dump_row, lane, set, merge, i0, epi_s, negp, one);
            else emit_lanes<K, OutT, false, BANDS, SKEW, SKEW || FPQ>(A, dump_row, lane, set, merge, i0, epi_s);
        }

        it = itn;
        ec = en;
        itn = __shfl_sync(0xffffffffu, itnn, 0);
        en = load_vset(A, itn, n_vsets, f);
    }
    if (__any_sync(0xffffffffu, maxid >= p) && lane == 0 && A.status) atomicOr(A.status, MHB_STATUS_ID_GE_PRIME);
}

// ----------------------------------------------------------------------------
// Small batches (n_sets <= kSmallPlan): latency-shaped kernel
// ----------------------------------------------------------------------------
//
// cfg1 (10,000 sets, N = 128) has ~1,250 warp items for 2,368 warp slots, so the
// large-batch kernel's static item -> warp map left half the slots idle and put two
// items on scheduler 0 of every SM (warps 0 and 4 of a CTA share an SMSP) while the
// others ran one: the kernel took 2x its ALU time.  Here
//   * every set is cut into Q contiguous parts (Q = 1, 2, 4): Q threads walk one
//     (set, lane block) and meet in a shuffle min, so there are Q x more, Q x shorter
//     items;
//   * each CTA owns a contiguous range of items and its warps claim them from a
//     shared-memory counter, so the 2 warps per SMSP of a CTA balance each other;
//   * the Q threads of a (set, lane block) split its epilogue quads;
//   * the plan kernel zeroes the caller's status word and the sign kernel ORs into it
//     (no last-CTA copy), and the last-CTA finalize runs only when the plan found long
//     sets (n_big > 0): no fence or atomic round trips at the end of a typical batch.
struct SmallArgs {
    int32_t* status_out;  // the caller's status word (zeroed by plan_small_kernel), or null
    int32_t log2Q;        // parts per (set, lane block)
};

template <int K, typename OutT>
__device__ __forceinline__ void emit_quads(const SignArgs& A, const uint32_t* dump_row, int lane, int64_t set,
                                           bool merge, int64_t i0, const InvTab* epi_s, bool epi_smem, int qlo,
                                           int qhi) {
    constexpr int NQ = K / 4;
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;
    const uint32_t p = A.p;
    const int32_t N = A.n_hash;
    const bool vec_ok = (N & 3) == 0;
    OutT* row = reinterpret_cast<OutT*>(A.out) + set * (int64_t)N;
#pragma unroll 1
    for (int q = qlo; q < qhi; ++q) {
        const int64_t i = i0 + 4 * q;
        if (i >= N) break;
        const uint4 m = *reinterpret_cast<const uint4*>(dump_row + ((q ^ (lane & SWZ)) << 2));
        const uint32_t h[4] = {m.x, m.y, m.z, m.w};
        if (merge) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (i + e < N) atomic_min_out(row + i + e, h[e]);
            continue;
        }
        uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t ie = min(i + e, A.n_tot - 1);
            const InvTab t = epi_smem ? epi_s[ie] : A.inv[ie];
            x[e] = invert_entry(t, h[e], p);
        }
        if (vec_ok && i + 3 < N) {
            store4(row + i, x[0], x[1], x[2], x[3]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (i + e < N) row[i + e] = (OutT)x[e];
        }
    }
}

// Ids of a warp item staged in shared memory: an item's sets are consecutive virtual
// sets, so their features are ONE contiguous range of ids.  Each warp copies the range of
// its next item while it walks the current one (double buffer): the 16-byte-aligned
// middle of the range with one TMA bulk copy (cp.async.bulk, completion counted on a
// per-buffer mbarrier), the < 4 ids at each unaligned end with 4-byte cp.async.
// ids per buffer (wider items walk from global memory); K = 64 takes half, so that
// two CTAs still fit an SM next to its 64 KB of dump rows.  A buffer holds 4 more
// (the range starts at its global address's offset within 16 bytes).
__host__ __device__ constexpr int stage_ids(int K) { return K >= 64 ? 256 : 512; }
#ifndef MHB_STAGE_TMA
#define MHB_STAGE_TMA 0  // 1: the middle by one TMA bulk copy + mbarrier (cfg1 kernel 23.9 us vs 22.7 with cp.async)
#endif
__host__ __device__ constexpr int stage_stride(int K) { return stage_ids(K) + 4; }

__device__ __forceinline__ void cp_async4(uint32_t saddr, const uint32_t* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
}
// One thread: expect `bytes` on the barrier, then the bulk copy that delivers them.
__device__ __forceinline__ void tma_load_1d(uint32_t sdst, const void* gsrc, uint32_t bytes, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sdst), "l"(gsrc), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P;\n"
                 "MHB_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                 "@!P bra MHB_WAIT_%=;\n\t}" ::"r"(mbar), "r"(parity) : "memory");
}

template <int K, bool ITER, bool NARROW, typename OutT, bool FPQ = false>
__global__ void __maxnreg__(128) sign_small_batch_kernel(SignArgs A, uint32_t p, uint32_t bpar, uint32_t negp, uint32_t one, SmallArgs SA) {
    constexpr int kStageIds_ = stage_ids(K);
    constexpr int kStride = stage_stride(K);
    extern __shared__ uint4 smem_raw[];
    __shared__ unsigned s_next;
    __shared__ int s_last;
    __shared__ __align__(8) unsigned long long s_mbar[kBlock / 32][2];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* dump_row = reinterpret_cast<uint32_t*>(smem_raw) + (warp * 32 + lane) * K;
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem_raw) + kBlock * K + warp * 2 * kStride;
    InvTab* epi_s = reinterpret_cast<InvTab*>(reinterpret_cast<uint32_t*>(smem_raw) + kBlock * K +
                                              (kBlock / 32) * 2 * kStride);
    const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(&s_mbar[warp][0]);
    if (lane == 0) {
        mbar_init(mbar0);
        mbar_init(mbar0 + 8);
        // make the initialised barriers visible to the async (TMA) proxy
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int log2Q = SA.log2Q;
    const int Q = 1 << log2Q;
    const int F = A.F;
    const int g = lane >> A.log2F;
    const int f = lane & (F - 1);
    const int jset = f >> log2Q;         // set slot of the warp group
    const int part = f & (Q - 1);        // part of the set this thread walks
    const int log2Fs = A.log2F - log2Q;  // sets per warp group = F / Q

    // launched with programmatic stream serialization (PDL): this grid may start while
    // plan_small_kernel finishes; everything below reads the plan's outputs
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the plan's counts and the epilogue table load together, before the one barrier
    const unsigned long long n_vsets = *((volatile unsigned long long*)&A.sched->n_vsets);
    const unsigned long long n_big = *((volatile unsigned long long*)&A.sched->n_big);
    const bool epi_smem = A.n_tot <= kEpiSmemLanes;
    if (epi_smem)
        for (int i = threadIdx.x; i < A.n_tot; i += blockDim.x) epi_s[i] = A.inv[i];
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();

    const unsigned long long n_groups = (n_vsets + (1ull << log2Fs) - 1) >> log2Fs;
    const unsigned long long n_items = n_groups * (unsigned)A.n_super;
    const unsigned long long per = (n_items + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = per * blockIdx.x;
    const unsigned long long hi = min(lo + per, n_items);

    auto claim = [&]() -> unsigned long long {
        unsigned v = 0;
        if (lane == 0) v = atomicAdd(&s_next, 1u);
        return lo + __shfl_sync(0xffffffffu, v, 0);
    };
    auto vset_of = [&](unsigned long long it) -> VSet {
        VSet v;
        v.f0 = 0;
        v.meta = -1;
        if (it < hi) {
            const unsigned long long group = A.n_super == 1 ? it : it / (unsigned)A.n_super;
            const unsigned long long k = (group << log2Fs) + jset;
            if (k < n_vsets) v = A.vsets[k];
        }
        return v;
    };
    // The item's id range [r0, r0 + width): slot 0 (lane 0) holds its first virtual set.
    // Staged (width <= kStageIds_) into buffer b: buffer index k holds id r0 - pad + k,
    // pad = r0's 4-byte offset within its 16-byte line, so buffer and global 16-byte
    // boundaries coincide.  The aligned middle goes by TMA (lane 0; `tma` = issued), the
    // ends by cp.async (one commit group per item, even when empty).
    auto stage_item = [&](const VSet& v, int b, long long& r0, int& pad, bool& tma) -> bool {
        r0 = __shfl_sync(0xffffffffu, v.f0, 0);
        const unsigned end = v.meta >= 0 ? (unsigned)(v.f0 + (v.meta & 2047) + 1 - r0) : 0u;
        const unsigned width = __reduce_max_sync(0xffffffffu, end);
        const bool staged = width > 0 && width <= (unsigned)kStageIds_;
        tma = false;
        pad = 0;
        if (staged) {
            const uint32_t* g0 = A.ids + r0;
            pad = (int)(((uintptr_t)g0 >> 2) & 3);
            const uint32_t* gb = g0 - pad;  // 16-byte aligned; buffer index 0
            const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(stage + b * kStride);
            const int k0 = pad, k1 = pad + (int)width;     // buffer range of the item
            const int m0 = (k0 + 3) & ~3, m1 = k1 & ~3;    // aligned middle [m0, m1)
            const int h1 = min(m0, k1);                    // head [k0, h1)
            const int t0 = max(m1, h1);                    // tail [t0, k1)
            const int nh = h1 - k0, nt = k1 - t0;
            if (lane < nh) cp_async4(sbuf + 4 * (k0 + lane), gb + k0 + lane);
            else if (lane >= 8 && lane < 8 + nt) cp_async4(sbuf + 4 * (t0 + lane - 8), gb + t0 + lane - 8);
            if (m1 > m0) {
#if MHB_STAGE_TMA
                tma = true;
                // the buffer's previous contents were read through the generic proxy
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    tma_load_1d(sbuf + 4 * m0, gb + m0, 4u * (uint32_t)(m1 - m0), mbar0 + 8 * b);
                }
#else
                for (int k = m0 + 4 * lane; k < m1; k += 128) cp_async16(sbuf + 4 * k, gb + k);
#endif
            }
        }
        cp_async_commit();
        return staged;
    };

    uint32_t phase = 0;  // bit b: parity of buffer b's barrier for its next completion
    unsigned long long it = claim();
    VSet ec = vset_of(it);
    int cur = 0;
    long long r0c;
    int padc;
    bool tmac;
    bool stc = stage_item(ec, 0, r0c, padc, tmac);

    LaneState<K, ITER> ls;
    ls.negp = negp;
    ls.one = one;
    int cur_sb = -1;
    uint32_t maxid = 0;

    while (it < hi) {  // uniform: lane 0's claim, broadcast
        // the next item's ids go into the other buffer while this one is walked
        const unsigned long long itn = claim();
        const VSet en = vset_of(itn);
        long long r0n;
        int padn;
        bool tman;
        const bool stn = stage_item(en, cur ^ 1, r0n, padn, tman);

        int sb = 0;
        if (A.n_super > 1) sb = (int)(it % (unsigned)A.n_super);
        if (sb != cur_sb) {
            const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
            if constexpr (ITER) {
                const LaneTab t = A.tab[i0];
                ls.tA = t.A; ls.tAp = t.Ap; ls.tB = t.B;
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const LaneTab t = A.tab[i0 + k];
                    ls.cA[k] = t.A; ls.cAp[k] = t.Ap; ls.cB[k] = t.B;
                }
            }
            cur_sb = sb;
        }
        // this thread's part [s0, s0 + n) of its virtual set (parts past the end repeat
        // the last feature, harmless for a minimum; idle slots walk ids[0])
        const bool valid = ec.meta >= 0;
        int n = 1;
        const uint32_t* base = A.ids;
        if (valid) {
            const int nv = (int)(ec.meta & 2047) + 1;
            const int c = (nv + Q - 1) >> log2Q;
            const int s0 = min(part * c, nv - 1);
            n = max(min(s0 + c, nv) - s0, 1);
            base = stc ? stage + cur * kStride + padc + (ec.f0 - r0c) + s0 : A.ids + ec.f0 + s0;
        } else if (stc) {
            base = stage + cur * kStride + padc;
        }
        cp_async_wait1();  // this item's end copies (the next item's may still be in flight)
        if (tmac) {         // and its TMA middle
            mbar_wait(mbar0 + 8 * cur, (phase >> cur) & 1u);
            phase ^= 1u << cur;
        }
        __syncwarp();
        const int last = n - 1;
        const int n_max = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
        const int rounds = (n_max + 1) >> 1;
        const bool odd = n_max & 1;

        uint32_t best[K];
        uint32_t xa = base[0], xb = base[min(1, last)];
        if (rounds == 1) {
            maxid = __vimax3_u32(maxid, xa, xb);
            round2<K, ITER, NARROW, true, FPQ>(best, ls, xa, xb, p, bpar);
        } else {
            uint32_t pa = base[min(2, last)], pb = base[min(3, last)];
            maxid = __vimax3_u32(maxid, xa, xb);
            round2<K, ITER, NARROW, true, FPQ>(best, ls, xa, xb, p, bpar);
            xa = pa; xb = pb;
            int o = 4;
#pragma unroll 1
            for (int r = 1; r + 1 < rounds; ++r, o += 2) {
                pa = base[min(o, last)];
                pb = base[min(o + 1, last)];
                maxid = __vimax3_u32(maxid, xa, xb);
                round2<K, ITER, NARROW, false, FPQ>(best, ls, xa, xb, p, bpar);
                xa = pa; xb = pb;
            }
            if (odd) {
                maxid = max(maxid, xa);
                round1<K, ITER, NARROW, FPQ>(best, ls, xa, p, bpar);
            } else {
                maxid = __vimax3_u32(maxid, xa, xb);
                round2<K, ITER, NARROW, false, FPQ>(best, ls, xa, xb, p, bpar);
            }
        }
        // the Q parts of a (set, lane block) meet: afterwards every part holds the minima
        for (int o = 1; o < Q; o <<= 1) {
#pragma unroll
            for (int k = 0; k < K; ++k) best[k] = min(best[k], __shfl_xor_sync(0xffffffffu, best[k], o));
        }
        if (valid) {
            const int64_t set = ec.meta >> 12;
            const bool merge = (ec.meta >> 11) & 1;
            const int64_t i0 = (int64_t)sb * A.L + (int64_t)g * K;
            dump_best<K>(best, dump_row, lane);
            constexpr int NQ = K / 4;
            emit_quads<K, OutT>(A, dump_row, lane, set, merge, i0, epi_s, epi_smem, (part * NQ) >> log2Q,
                                ((part + 1) * NQ) >> log2Q);
        }
        __syncwarp();  // every lane is done with this buffer before it is restaged
        it = itn;
        ec = en;
        r0c = r0n;
        padc = padn;
        tmac = tman;
        stc = stn;
        cur ^= 1;
    }
    if (__any_sync(0xffffffffu, maxid >= p) && lane == 0 && SA.status_out)
        atomicOr(SA.status_out, MHB_STATUS_ID_GE_PRIME);
    if (blockIdx.x == 0 && threadIdx.x == 0 && SA.status_out) {
        const int32_t plan_status = *((volatile int32_t*)&A.sched->status);  // empty sets, bad parameters
        if (plan_status) atomicOr(SA.status_out, plan_status);
    }
    if (n_big == 0) return;
    // long sets: the last CTA to finish inverts their merged rows
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&A.sched->done, 1ull) == (unsigned long long)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        finalize_rows<OutT>(A, 0, 1);
    }
}

template <typename OutT>
__global__ void finalize_kernel(SignArgs A) {
    finalize_rows<OutT>(A, blockIdx.x, gridDim.x);
}

// ----------------------------------------------------------------------------
// Host launch
// ----------------------------------------------------------------------------

// Optional per-launch timing of the main kernel: CUDA events recorded on the
// launch stream right before and after it (mhb_profile_begin / _end).
namespace {
std::mutex g_prof_mu;
bool g_prof_on = false;
int g_prof_cap = 0, g_prof_n = 0, g_prof_dev = -1;
cudaEvent_t* g_prof_ev = nullptr;
}  // namespace

using SignKernelFn = void (*)(SignArgs, uint32_t, uint32_t, uint32_t, uint32_t);

template <bool ITER, bool NARROW, typename OutT>
static SignKernelFn pick_kernel(int K) {
    switch (K) {
        case 8: return sign_kernel<8, ITER, NARROW, OutT>;
        case 16: return sign_kernel<16, ITER, NARROW, OutT>;
        case 32: return sign_kernel<32, ITER, NARROW, OutT>;
        default: break;
    }
    if constexpr (ITER) return sign_kernel<64, ITER, NARROW, OutT>;
    return nullptr;
}

// Iterative K = 64 with G >= 16 lane groups (N >= 1024): the skewed epilogue table.
static SignKernelFn select_skew_kernel(bool narrow, int out_dtype) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (narrow) return i64 ? sign_kernel<64, true, true, long long, false, false, true>
                           : sign_kernel<64, true, true, uint32_t, false, false, true>;
    return i64 ? sign_kernel<64, true, false, long long, false, false, true>
               : sign_kernel<64, true, false, uint32_t, false, false, true>;
}

static SignKernelFn select_fpq_kernel(int out_dtype, int K) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (K == 16) return i64 ? sign_kernel<16, false, true, long long, false, true>
                            : sign_kernel<16, false, true, uint32_t, false, true>;
    if (K == 8) return i64 ? sign_kernel<8, false, true, long long, false, true>
                           : sign_kernel<8, false, true, uint32_t, false, true>;
    return nullptr;
}

static SignKernelFn select_bands_kernel(bool narrow, int out_dtype, int K, bool skew) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (K == 64 && skew) {  // N >= 1024: the skewed epilogue table (cfg4: 128 bands x 16 rows)
        if (narrow) return i64 ? sign_kernel<64, true, true, long long, true, false, true>
                               : sign_kernel<64, true, true, uint32_t, true, false, true>;
        return i64 ? sign_kernel<64, true, false, long long, true, false, true>
                   : sign_kernel<64, true, false, uint32_t, true, false, true>;
    }
    if (K == 64) {
        if (narrow) return i64 ? sign_kernel<64, true, true, long long, true> : sign_kernel<64, true, true, uint32_t, true>;
        return i64 ? sign_kernel<64, true, false, long long, true> : sign_kernel<64, true, false, uint32_t, true>;
    }
    if (K == 32) {
        if (narrow) return i64 ? sign_kernel<32, true, true, long long, true> : sign_kernel<32, true, true, uint32_t, true>;
        return i64 ? sign_kernel<32, true, false, long long, true> : sign_kernel<32, true, false, uint32_t, true>;
    }
    return nullptr;
}

static SignKernelFn select_kernel(int kind, bool narrow, int out_dtype, int K) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (kind == KIND_ITERATIVE) {
        if (narrow) return i64 ? pick_kernel<true, true, long long>(K) : pick_kernel<true, true, uint32_t>(K);
        return i64 ? pick_kernel<true, false, long long>(K) : pick_kernel<true, false, uint32_t>(K);
    }
    if (narrow) return i64 ? pick_kernel<false, true, long long>(K) : pick_kernel<false, true, uint32_t>(K);
    return i64 ? pick_kernel<false, false, long long>(K) : pick_kernel<false, false, uint32_t>(K);
}

using SmallKernelFn = void (*)(SignArgs, uint32_t, uint32_t, uint32_t, uint32_t, SmallArgs);

template <bool ITER, bool NARROW, typename OutT>
static SmallKernelFn pick_small(int K) {
    switch (K) {
        case 8: return sign_small_batch_kernel<8, ITER, NARROW, OutT>;
        case 16: return sign_small_batch_kernel<16, ITER, NARROW, OutT>;
        default: break;
    }
    // the random family keeps K <= 16 (three constants per lane in registers)
    if constexpr (ITER) return K == 32 ? sign_small_batch_kernel<32, ITER, NARROW, OutT>
                                       : sign_small_batch_kernel<64, ITER, NARROW, OutT>;
    return nullptr;
}

static SmallKernelFn select_small_kernel(int kind, bool narrow, int out_dtype, int K, bool fpq) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (fpq) {
        if (K == 16) return i64 ? sign_small_batch_kernel<16, false, true, long long, true>
                                : sign_small_batch_kernel<16, false, true, uint32_t, true>;
        if (K == 8) return i64 ? sign_small_batch_kernel<8, false, true, long long, true>
                               : sign_small_batch_kernel<8, false, true, uint32_t, true>;
        return nullptr;
    }
    if (kind == KIND_ITERATIVE) {
        if (narrow) return i64 ? pick_small<true, true, long long>(K) : pick_small<true, true, uint32_t>(K);
        return i64 ? pick_small<true, false, long long>(K) : pick_small<true, false, uint32_t>(K);
    }
    if (narrow) return i64 ? pick_small<false, true, long long>(K) : pick_small<false, true, uint32_t>(K);
    return i64 ? pick_small<false, false, long long>(K) : pick_small<false, false, uint32_t>(K);
}

// Parts per (set, lane block) for the small-batch kernel: enough items for about two
// per warp slot (the CTAs' shared counters then balance their SMSPs), but parts of at
// least ~8 features.  MHB_SMALL_Q forces it (tuning).
static int pick_parts(int64_t n_sets, int64_t nnz, const Geometry& geo, int sms, int occ) {
    static const int forced = [] {
        const char* e = std::getenv("MHB_SMALL_Q");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2 || forced == 4) return forced <= geo.F ? forced : geo.F;
    const int64_t items = (n_sets + geo.F - 1) / geo.F * geo.n_super;
    const int64_t slots = (int64_t)sms * occ * (kBlock / 32);
    const int64_t mean = n_sets > 0 ? nnz / n_sets : 0;
    int Q = 1;
    while (Q < 4 && Q < geo.F && items * Q < 2 * slots && mean / (2 * Q) >= 8) Q *= 2;
    return Q;
}

// Occupancy (CTAs per SM) per (kernel, device, dynamic smem); computed once.  The
// dynamic-smem limit is raised to the device maximum the first time a kernel is seen.
static int blocks_per_sm(const void* fn, size_t smem, const DeviceInfo& dev) {
    static std::mutex mu;
    struct Entry { const void* fn; int dev; size_t smem; int occ; };
    static Entry cache[512];
    static int n_cache = 0;
    std::lock_guard<std::mutex> lock(mu);
    bool seen = false;
    for (int i = 0; i < n_cache; ++i) {
        if (cache[i].fn == (const void*)fn && cache[i].dev == dev.device) {
            seen = true;
            if (cache[i].smem == smem) return cache[i].occ;
        }
    }
    if (!seen) {
        // the dynamic limit is what the opt-in maximum leaves after the kernel's static smem
        cudaFuncAttributes fa{};
        size_t stat = 0;
        if (cudaFuncGetAttributes(&fa, (const void*)fn) == cudaSuccess) stat = fa.sharedSizeBytes;
        cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(dev.smem_optin > stat ? dev.smem_optin - stat : 0));
        cudaGetLastError();
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kBlock, smem) != cudaSuccess)
        occ = 1;
    if (occ < 1) occ = 1;
    if (n_cache < 512) cache[n_cache++] = Entry{(const void*)fn, dev.device, smem, occ};
    return occ;
}

int check_sign_params(int kind, uint64_t a, uint64_t b, bool have_random_arrays, uint64_t prime, int32_t n_hash) {
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function, got %d", n_hash);
    if (prime < 3 || !is_prime_u64(prime)) return set_error(MHB_ERR_INVALID, "modulus %llu is not prime",
                                                             (unsigned long long)prime);
    if (prime >= (1ull << 63))
        return set_error(MHB_ERR_UNSUPPORTED, "prime %llu >= 2^63 is out of range", (unsigned long long)prime);
    if (prime >= (1ull << 31) && kind == KIND_RANDOM)
        return set_error(MHB_ERR_UNSUPPORTED,
                         "prime %llu >= 2^31: random-family parameters need 64 bits, use mhb_sign_random_csr_u64",
                         (unsigned long long)prime);
    if (kind == KIND_ITERATIVE) {
        if (a < 1 || a >= prime || b >= prime)
            return set_error(MHB_ERR_INVALID, "need 1 <= a < p and 0 <= b < p");
        if (a + (uint64_t)n_hash >= prime)
            return set_error(MHB_ERR_INVALID,
                             "need a + size < prime to keep every member invertible; got a=%llu, size=%d, "
                             "prime=%llu", (unsigned long long)a, n_hash, (unsigned long long)prime);
    } else if (!have_random_arrays) {
        return set_error(MHB_ERR_INVALID, "random family needs device arrays a and b");
    }
    return MHB_OK;
}

int launch_sign(int kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t nnz,
                uint64_t a, uint64_t b, const uint32_t* ra, const uint32_t* rb, uint64_t prime,
                int32_t n_hash, void* out, int32_t out_dtype, int32_t* status, void* workspace,
                size_t workspace_bytes, cudaStream_t st, unsigned long long* keys, int32_t rows_per_band,
                int32_t write_sig) {
    clear_error();
    if (n_sets < 0 || nnz < 0) return set_error(MHB_ERR_INVALID, "n_sets and nnz must be >= 0");
    if (out_dtype != MHB_OUT_U32 && out_dtype != MHB_OUT_I64)
        return set_error(MHB_ERR_INVALID, "unknown out_dtype %d", out_dtype);
    if (int rc = check_sign_params(kind, a, b, ra != nullptr && rb != nullptr, prime, n_hash)) return rc;
    const bool wide = prime >= (1ull << 31);
    if (n_sets > 0 && (indptr == nullptr || out == nullptr))
        return set_error(MHB_ERR_INVALID, "null indptr/out");
    if (nnz > 0 && ids == nullptr) return set_error(MHB_ERR_INVALID, "null ids");
    if (n_sets >= (1ll << 51)) return set_error(MHB_ERR_INVALID, "too many sets");

    if (wide)  // 64-bit residues; no workspace needed
        return launch_sign_wide(true, indptr, ids, n_sets, a, b, nullptr, nullptr, prime, n_hash, out, out_dtype,
                                status, st);

    const WorkspaceLayout wl = workspace_layout(n_sets, nnz, n_hash);
    if (workspace == nullptr || workspace_bytes < wl.total)
        return set_error(MHB_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", wl.total,
                         workspace_bytes);

    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    const Geometry geo = choose_geometry(kind, n_hash, pick_lanes(kind, n_hash, n_sets, dev.sms, keys != nullptr));
    char* ws = static_cast<char*>(workspace);
    SignArgs A{};
    A.indptr = indptr;
    A.ids = ids;
    A.n_sets = n_sets;
    A.p = (uint32_t)prime;
    A.b = (uint32_t)b;
    A.ia = a;
    A.n_hash = n_hash;
    A.F = geo.F;
    A.log2F = geo.log2F;
    A.n_super = geo.n_super;
    A.L = geo.L;
    A.K = geo.K;
    A.n_tot = geo.n_tot;
    A.kind = kind;
    A.tab = reinterpret_cast<LaneTab*>(ws + wl.tab);
    A.inv = reinterpret_cast<InvTab*>(ws + wl.inv);
    A.sched = reinterpret_cast<Sched*>(ws + wl.sched);
    A.hist = reinterpret_cast<unsigned*>(ws + wl.hist);
    A.big = reinterpret_cast<int64_t*>(ws + wl.big);
    A.vsets = reinterpret_cast<VSet*>(ws + wl.vsets);
    A.status = status;
    A.out = out;
    A.ra = ra;
    A.rb = rb;
    A.keys = keys;
    A.rows = rows_per_band;
    A.write_sig = write_sig;
    A.chunk = choose_chunk(n_sets, nnz, n_hash);

    // keys (fused band epilogue) have no small-batch instances: they keep the sorted plan
    // the enumerating kernel (gap.cu) where its cost model prefers it (gap_wanted); the
    // rest of the batches of <= kSmallPlan sets keep the one-launch small-batch plan
    const bool gap = keys == nullptr && gap_wanted(kind, prime, n_hash, n_sets, nnz);
    const bool small_plan = n_sets > 0 && n_sets <= kSmallPlan && keys == nullptr && !gap;
    // sched and hist are contiguous at the start of the workspace (zeroed: the sorted
    // plan's histogram, or the small plan's look-back state)
    rc = cuda_check(cudaMemsetAsync(ws, 0, wl.tab, st), "memset plan state");
    if (rc) return rc;
    int32_t* status_out = nullptr;
    if (small_plan && status) {
        // no status memset: plan_small_kernel zeroes *status and ORs its flags into the
        // (zeroed) workspace word; sign_small_batch_kernel ORs both into *status
        A.status = &A.sched->status;
        status_out = status;
    } else if (status) {
        rc = cuda_check(cudaMemsetAsync(status, 0, sizeof(int32_t), st), "memset status");
        if (rc) return rc;
    }
    if (n_sets == 0) return MHB_OK;

    // random family with p <= 2^23: float-quotient lanes (walk2_random_fpq); the plan
    // kernels build their lane tables, so the flag is set before they launch
    const bool fpq = !keys && kind == KIND_RANDOM && prime <= (1ull << 23) && (geo.K == 16 || geo.K == 8);
    A.fpq = fpq ? 1 : 0;

    if (small_plan) {
        // tiles of sets, then CTAs for the lane tables (N may be 10^5)
        const int64_t lane_ctas = std::min<int64_t>((geo.n_tot + kSmallTile - 1) / kSmallTile, (int64_t)dev.sms * 4);
        const int64_t tiles = (n_sets + kSmallTile - 1) / kSmallTile + lane_ctas;
        if (out_dtype == MHB_OUT_I64)
            plan_small_kernel<long long><<<(unsigned)tiles, kSmallTile, 0, st>>>(A, status_out);
        else
            plan_small_kernel<uint32_t><<<(unsigned)tiles, kSmallTile, 0, st>>>(A, status_out);
        rc = cuda_check(cudaGetLastError(), "plan_small launch");
        if (rc) return rc;
    } else {
        int64_t work = n_sets > geo.n_tot ? n_sets : geo.n_tot;
        int64_t blocks = (work + 255) / 256;
        int64_t cap = (int64_t)dev.sms * 4;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        if (out_dtype == MHB_OUT_I64)
            plan_count_kernel<long long><<<(unsigned)blocks, 256, 0, st>>>(A);
        else
            plan_count_kernel<uint32_t><<<(unsigned)blocks, 256, 0, st>>>(A);
        if (gap) {
            // gap.cu: the lane tables are all it needs of the plan
            rc = cuda_check(cudaGetLastError(), "plan_count launch");
            if (rc) return rc;
            int prof_slot = -1;
            {
                std::lock_guard<std::mutex> lock(g_prof_mu);
                if (g_prof_on && g_prof_n < g_prof_cap && g_prof_dev == dev.device) prof_slot = g_prof_n++;
            }
            if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot], st);
            rc = launch_sign_gap(A, nnz, out_dtype, dev, st);
            if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot + 1], st);
            return rc;
        }
        plan_scan_kernel<<<1, kChunk, 0, st>>>(A);
        int64_t sblocks = (n_sets + 1023) / 1024;
        if (sblocks > (int64_t)dev.sms * 4) sblocks = (int64_t)dev.sms * 4;
        if (sblocks < 1) sblocks = 1;
        if (out_dtype == MHB_OUT_I64)
            plan_scatter_kernel<long long><<<(unsigned)sblocks, 256, 0, st>>>(A);
        else
            plan_scatter_kernel<uint32_t><<<(unsigned)sblocks, 256, 0, st>>>(A);
        rc = cuda_check(cudaGetLastError(), "plan kernels launch");
        if (rc) return rc;
    }

    const bool narrow = (3ull * prime) < (1ull << 32);
    const bool skew = kind == KIND_ITERATIVE && geo.K == 64 && geo.G >= 16;
    const size_t smem = (size_t)kBlock * geo.K * sizeof(uint32_t) +
                        (geo.n_tot <= kEpiSmemLanes ? (size_t)(geo.n_tot + geo.n_tot / geo.K + 1) * sizeof(InvTab) : 0) +
                        ((skew && (keys ? MHB_BV_STAGE : MHB_SV_STAGE)) || (fpq && MHB_RV_STAGE)
                             ? (size_t)kBlock / 32 * 2 * kSetStage * sizeof(uint32_t) : 0);
    const int64_t max_vsets = n_sets + nnz / A.chunk;
    const int64_t items_ub = ((max_vsets + geo.F - 1) / geo.F) * geo.n_super;
    // small batches (one-launch unsorted plan): sign_small_batch_kernel
    if (small_plan) {
        SmallKernelFn sfn = select_small_kernel(kind, narrow, out_dtype, geo.K, fpq);
        if (!sfn) return set_error(MHB_ERR_INVALID, "no small-batch kernel instance for K=%d", geo.K);
        const size_t ssmem = (size_t)kBlock * geo.K * sizeof(uint32_t) +
                             (size_t)(kBlock / 32) * 2 * stage_stride(geo.K) * sizeof(uint32_t) +
                             (geo.n_tot <= kEpiSmemLanes ? (size_t)geo.n_tot * sizeof(InvTab) : 0);
        const int occ = blocks_per_sm((const void*)sfn, ssmem, dev);
        const int Q = pick_parts(n_sets, nnz, geo, dev.sms, occ);
        SmallArgs SA{status_out, 0};
        while ((1 << SA.log2Q) < Q) ++SA.log2Q;
        // one CTA per 8 items (a warp each) up to the resident grid; a CTA's warps share
        // its item range through a shared-memory counter
        const int64_t items = (n_sets * Q + geo.F - 1) / geo.F * geo.n_super;
        int64_t blocks = (items + (kBlock / 32) - 1) / (kBlock / 32);
        const int64_t cap = (int64_t)occ * dev.sms;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        int prof_slot = -1;
        {
            std::lock_guard<std::mutex> lock(g_prof_mu);
            if (g_prof_on && g_prof_n < g_prof_cap && g_prof_dev == dev.device) prof_slot = g_prof_n++;
        }
        if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot], st);
        // programmatic dependent launch: the grid is set up while the plan kernel runs
        // (the kernel waits on griddepcontrol before its first read); MHB_PDL=0 turns it off
        static const bool pdl = [] {
            const char* e = std::getenv("MHB_PDL");
            return !(e && e[0] == '0');
        }();
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3(kBlock);
        cfg.dynamicSmemBytes = ssmem;
        cfg.stream = st;
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        rc = cuda_check(cudaLaunchKernelEx(&cfg, sfn, A, A.p, A.b, 0u - A.p, 1u, SA), "sign_small_batch_kernel launch");
        if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot + 1], st);
        return rc;
    }
    SignKernelFn fn = keys   ? select_bands_kernel(narrow, out_dtype, geo.K, skew)
                      : fpq  ? select_fpq_kernel(out_dtype, geo.K)
                      : skew ? select_skew_kernel(narrow, out_dtype)
                             : select_kernel(kind, narrow, out_dtype, geo.K);
    if (!fn) return set_error(MHB_ERR_INVALID, "no kernel instance for K=%d", geo.K);
    SignKernelFn occ_fn = fpq ? select_fpq_kernel(out_dtype, geo.K) : select_kernel(kind, narrow, out_dtype, geo.K);
    const int occ = blocks_per_sm((const void*)(keys || skew ? fn : occ_fn), smem, dev);
    int64_t blocks = (items_ub + (kBlock / 32) - 1) / (kBlock / 32);
    const int64_t cap = (int64_t)occ * dev.sms;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    int prof_slot = -1;
    {
        std::lock_guard<std::mutex> lock(g_prof_mu);
        if (g_prof_on && g_prof_n < g_prof_cap && g_prof_dev == dev.device) prof_slot = g_prof_n++;
    }
    if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot], st);
    fn<<<(unsigned)blocks, kBlock, smem, st>>>(A, A.p, A.b, 0u - A.p, 1u);
    if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot + 1], st);
    rc = cuda_check(cudaGetLastError(), "sign_kernel launch");
    if (rc) return rc;

    {
        // warps loop over long-set rows (finalize_rows); up to 16 blocks of 8 warps per SM
        // hide the row loads, and a batch without long sets pays for few empty blocks
        int64_t fb = (nnz / (A.chunk + 1) + 7) / 8;
        if (fb > (int64_t)dev.sms * 16) fb = (int64_t)dev.sms * 16;
        if (fb < 1) fb = 1;
        if (out_dtype == MHB_OUT_I64)
            finalize_kernel<long long><<<(unsigned)fb, 256, 0, st>>>(A);
        else
            finalize_kernel<uint32_t><<<(unsigned)fb, 256, 0, st>>>(A);
        rc = cuda_check(cudaGetLastError(), "finalize_kernel launch");
        if (rc) return rc;
    }
    return MHB_OK;
}

}  // namespace mhb

extern "C" int mhb_profile_begin(int32_t max_launches) {
    using namespace mhb;
    clear_error();
    std::lock_guard<std::mutex> lock(g_prof_mu);
    if (max_launches < 1) return set_error(MHB_ERR_INVALID, "max_launches must be >= 1");
    int dev = 0;
    int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    if (g_prof_ev) {
        cudaSetDevice(g_prof_dev);
        for (int i = 0; i < 2 * g_prof_cap; ++i) cudaEventDestroy(g_prof_ev[i]);
        delete[] g_prof_ev;
        g_prof_ev = nullptr;
        cudaSetDevice(dev);
    }
    g_prof_ev = new cudaEvent_t[2 * (size_t)max_launches];
    for (int i = 0; i < 2 * max_launches; ++i) {
        rc = cuda_check(cudaEventCreate(&g_prof_ev[i]), "cudaEventCreate");
        if (rc) return rc;
    }
    g_prof_cap = max_launches;
    g_prof_n = 0;
    g_prof_dev = dev;
    g_prof_on = true;
    return MHB_OK;
}

extern "C" int mhb_profile_end(float* total_ms, int32_t* n_launches) {
    using namespace mhb;
    clear_error();
    std::lock_guard<std::mutex> lock(g_prof_mu);
    g_prof_on = false;
    float sum = 0.f;
    for (int i = 0; i < g_prof_n; ++i) {
        int rc = cuda_check(cudaEventSynchronize(g_prof_ev[2 * i + 1]), "profile event sync");
        if (rc) return rc;
        float ms = 0.f;
        rc = cuda_check(cudaEventElapsedTime(&ms, g_prof_ev[2 * i], g_prof_ev[2 * i + 1]), "elapsed");
        if (rc) return rc;
        sum += ms;
    }
    if (total_ms) *total_ms = sum;
    if (n_launches) *n_launches = g_prof_n;
    g_prof_n = 0;
    return MHB_OK;
}

extern "C" int32_t mhb_sign_iterative_path(int64_t n_sets, int64_t nnz, uint64_t prime, int32_t n_hash) {
    return mhb::gap_wanted(mhb::KIND_ITERATIVE, prime, n_hash, n_sets, nnz) ? 1 : 0;
}

extern "C" size_t mhb_sign_workspace_bytes(int64_t n_sets, int64_t nnz, int32_t n_hash) {
    if (n_hash < 1) n_hash = 1;
    return mhb::workspace_layout(n_sets, nnz, n_hash).total;
}

extern "C" int mhb_sign_iterative_csr(const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
                                      int64_t nnz, uint64_t a, uint64_t b, uint64_t prime,
                                      int32_t n_hash, void* out, int32_t out_dtype, int32_t* status,
                                      void* workspace, size_t workspace_bytes, void* stream) {
    return mhb::launch_sign(mhb::KIND_ITERATIVE, indptr, ids, n_sets, nnz, a, b, nullptr, nullptr,
                            prime, n_hash, out, out_dtype, status, workspace, workspace_bytes,
                            static_cast<cudaStream_t>(stream));
}

// Iterative signatures with LSH band keys fused into the epilogue.
extern "C" int mhb_sign_iterative_csr_bands(const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t nnz,
                                            uint64_t a, uint64_t b, uint64_t prime, int32_t n_hash,
                                            int32_t rows_per_band, unsigned long long* keys, void* out,
                                            int32_t out_dtype, int32_t write_signatures, int32_t* status,
                                            void* workspace, size_t workspace_bytes, void* stream) {
    using namespace mhb;
    clear_error();
    if (!keys) return set_error(MHB_ERR_INVALID, "keys output is required");
    if (rows_per_band < 4 || rows_per_band % 4 != 0 || n_hash % rows_per_band != 0)
        return set_error(MHB_ERR_INVALID, "rows_per_band must be a multiple of 4 dividing n_hash (got %d, %d)",
                         rows_per_band, n_hash);
    const Geometry geo = choose_geometry(KIND_ITERATIVE, n_hash);
    if ((geo.K != 64 && geo.K != 32) || geo.K % rows_per_band != 0 || prime >= (1ull << 31))
        return set_error(MHB_ERR_UNSUPPORTED,
                         "fused band keys need 32 <= n_hash, rows_per_band dividing %d and prime < 2^31; "
                         "use mhb_sign_iterative_csr + mhb_band_keys", geo.K);
    if (gap_wanted(KIND_ITERATIVE, prime, n_hash, n_sets, nnz)) {
        // where the enumerating kernel (gap.cu) is the faster signer, signatures first and
        // the keys from the stored rows (cfg4: 18.9 + 2.8 ms against 31.8 ms fused into
        // the visiting kernel); the keys are the same function of the signatures either way
        int rc = launch_sign(KIND_ITERATIVE, indptr, ids, n_sets, nnz, a, b, nullptr, nullptr, prime, n_hash, out,
                             out_dtype, status, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
        if (rc) return rc;
        return mhb_band_keys(out, out_dtype, n_sets, n_hash, rows_per_band, keys, stream);
    }
    return launch_sign(KIND_ITERATIVE, indptr, ids, n_sets, nnz, a, b, nullptr, nullptr, prime, n_hash, out,
                       out_dtype, status, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), keys,
                       rows_per_band, write_signatures ? 1 : 0);
}

extern "C" int mhb_sign_random_csr(const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
                                   int64_t nnz, const uint32_t* a, const uint32_t* b, uint64_t prime,
                                   int32_t n_hash, void* out, int32_t out_dtype, int32_t* status,
                                   void* workspace, size_t workspace_bytes, void* stream) {
    return mhb::launch_sign(mhb::KIND_RANDOM, indptr, ids, n_sets, nnz, 0, 0, a, b, prime, n_hash,
                            out, out_dtype, status, workspace, workspace_bytes,
                            static_cast<cudaStream_t>(stream));
}
