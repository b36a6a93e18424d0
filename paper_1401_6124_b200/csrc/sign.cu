// sign.cu -- MinHash signatures over CSR sets on sm_100a (both hash families).
//
// Reference semantics (arXiv 1401.6124 reference package):
//   sign_iterative  kernels.py:44-73   h_i(x) = ((a+i)x + i*b) mod p, walked as
//                                      h <- h + (x+b) mod p with one conditional subtract
//   sign_random     kernels.py:21-41   h_i(x) = (a_i x + b_i) mod p
//   output          minhash.py:91-110  argmin feature id per hash index
//
// Design:
//  * A warp owns one work item = (set, feature chunk <= kChunk, lane pass).  Its
//    32 threads form G lane groups x F feature slices (G*F = 32).  Thread (g,f)
//    keeps K running minima in registers for hash lanes i0 .. i0+K-1 and walks
//    features f, f+F, ... of the item, two at a time.
//  * Per (thread, feature) setup is one Shoup multiply: h_{i0}(x) = A_{i0} x + B_{i0}
//    with per-lane constants from a table built once per call.  Per visit the
//    iterative family costs IADD + VIADDMNMX + 1/2 VIMNMX3 (2.5 instructions);
//    the random family costs IMAD.HI + 2 IMAD + 2 VIADDMNMX + 1/2 VIMNMX3.
//  * Only the min HASH VALUE is tracked.  Every family member is a bijection on
//    [0,p) (families.py:82,141; reference test test_families.py:178-186), so the
//    argmin is recovered exactly once per entry: x = (h - B_i) * A_i^{-1} mod p.
//  * Slices are combined through a swizzled per-warp shared-memory tile; the
//    epilogue inverts and stores.  Sets longer than kChunk are split into chunks
//    that merge with atomicMin on the output row; a finalize pass inverts them.
//  * Work items are handed out by a global atomic counter (persistent grid),
//    long-set chunks first.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "common.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

// ----------------------------------------------------------------------------
// Geometry
// ----------------------------------------------------------------------------

static int next_pow2(int v) {
    int r = 1;
    while (r < v) r <<= 1;
    return r;
}

Geometry choose_geometry(int kind, int32_t n_hash) {
    Geometry g{};
    int K;
    if (kind == KIND_ITERATIVE) {
        K = n_hash >= 128 ? 64 : n_hash >= 32 ? 32 : n_hash >= 16 ? 16 : 8;
    } else {
        K = n_hash >= 64 ? 32 : n_hash >= 16 ? 16 : 8;
    }
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

WorkspaceLayout workspace_layout(int64_t n_sets, int64_t nnz, int32_t n_hash) {
    // Both families share one layout; size for the larger lane table.
    Geometry gi = choose_geometry(KIND_ITERATIVE, n_hash);
    Geometry gr = choose_geometry(KIND_RANDOM, n_hash);
    int64_t n_tot = gi.n_tot > gr.n_tot ? gi.n_tot : gr.n_tot;
    int n_super = gi.n_super > gr.n_super ? gi.n_super : gr.n_super;
    int64_t nnz_pos = nnz > 0 ? nnz : 0;
    int64_t max_big_sets = nnz_pos / (kChunk + 1);
    if (max_big_sets > n_sets) max_big_sets = n_sets;
    int64_t max_big = max_big_sets * n_super;
    int64_t max_extra = (nnz_pos / kChunk) * n_super;

    WorkspaceLayout w{};
    size_t off = 0;
    w.sched = off;  off = align_up(off + sizeof(Sched), 256);
    w.tab = off;    off = align_up(off + (size_t)n_tot * sizeof(LaneTab), 256);
    w.inv = off;    off = align_up(off + (size_t)n_tot * sizeof(InvTab), 256);
    w.big = off;    off = align_up(off + (size_t)(max_big > 0 ? max_big : 1) * sizeof(int64_t), 256);
    w.extra = off;  off = align_up(off + (size_t)(max_extra > 0 ? max_extra : 1) * sizeof(Extra), 256);
    w.total = off;
    return w;
}

// ----------------------------------------------------------------------------
// Setup: lane tables + long-set plan
// ----------------------------------------------------------------------------

template <typename OutT>
__global__ void setup_kernel(SignArgs A) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint32_t p = A.p;

    for (int64_t i = tid; i < A.n_tot; i += stride) {
        uint32_t w, c;
        if (A.kind == KIND_ITERATIVE) {
            // member i: multiplier a+i, offset i*b (families.py:124-131)
            w = (uint32_t)((A.ia + (uint64_t)i) % p);
            if (w == 0) w = 1;  // only reachable on padded lanes i >= n_hash
            c = (uint32_t)(((uint64_t)i % p) * (uint64_t)A.b % p);
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
        t.Ap = shoup_companion(w, p);
        t.B = c;
        t.pad = 0;
        A.tab[i] = t;
        InvTab v;
        v.B = c;
        v.inv = inv_mod(w, p);
        v.invp = shoup_companion(v.inv, p);
        v.pad = 0;
        A.inv[i] = v;
    }

    OutT* out = reinterpret_cast<OutT*>(A.out);
    for (int64_t s = tid; s < A.n_sets; s += stride) {
        const int64_t lo = A.indptr[s], hi = A.indptr[s + 1];
        const int64_t n = hi - lo;
        if (n <= 0) {
            if (A.status) atomicOr(A.status, MHB_STATUS_EMPTY_SET);
            continue;
        }
        if (n > kChunk) {
            const int64_t nch = (n + kChunk - 1) / kChunk;
            unsigned long long eb = atomicAdd(&A.sched->n_extra,
                                              (unsigned long long)((nch - 1) * A.n_super));
            unsigned long long bb = atomicAdd(&A.sched->n_big, (unsigned long long)A.n_super);
            for (int sb = 0; sb < A.n_super; ++sb) {
                A.big[bb + sb] = s * A.n_super + sb;
                for (int64_t c = 1; c < nch; ++c) {
                    Extra e;
                    e.set = s;
                    e.sb = sb;
                    e.chunk = (int32_t)c;
                    A.extra[eb++] = e;
                }
            }
            OutT* row = out + s * (int64_t)A.n_hash;
            for (int32_t i = 0; i < A.n_hash; ++i) row[i] = (OutT)(~0u);
        }
    }
}

// ----------------------------------------------------------------------------
// Main kernel
// ----------------------------------------------------------------------------

// Argmin recovery: x = (h - B_i) * A_i^{-1} mod p, from a staged epilogue table entry.
__device__ __forceinline__ uint32_t invert_entry(const InvTab& v, uint32_t h, uint32_t p) {
    uint32_t d = h - v.B;
    d = __viaddmin_u32(d, p, d);  // d in [0,p)
    return reduce_once(shoup_lazy(v.inv, v.invp, d, p), p);
}

__device__ __forceinline__ uint32_t invert_lane(const SignArgs& A, int64_t i, uint32_t h) {
    const InvTab v = A.inv[i];
    return invert_entry(v, h, A.p);
}

__device__ __forceinline__ void atomic_min_out(uint32_t* p, uint32_t v) { atomicMin(p, v); }
__device__ __forceinline__ void atomic_min_out(long long* p, uint32_t v) {
    atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
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
// FIRST: the item's first round initialises best instead of folding into it.
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

template <int K, bool FIRST>
__device__ __forceinline__ void walk1_iter(uint32_t (&best)[K], uint32_t ha, uint32_t da, uint32_t p) {
    const uint32_t da2 = reduce_once(da + da, p);
#pragma unroll
    for (int k = 0; k < K; k += 2) {
        const uint32_t ga = reduce_once(ha + da, p);
        if (FIRST) {
            best[k] = ha;
            best[k + 1] = ga;
        } else {
            best[k] = min(best[k], ha);
            best[k + 1] = min(best[k + 1], ga);
        }
        if (k + 2 < K) ha = reduce_once(ha + da2, p);
    }
}

template <int K, bool NARROW, bool FIRST>
__device__ __forceinline__ void walk2_random(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                             const uint32_t (&cAp)[K], const uint32_t (&cB)[K],
                                             uint32_t xa, uint32_t xb, uint32_t p) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        uint32_t ra, rb;
        if (NARROW) {
            ra = mul_add_mod_narrow(cA[k], cAp[k], cB[k], xa, p);
            rb = mul_add_mod_narrow(cA[k], cAp[k], cB[k], xb, p);
        } else {
            ra = mul_add_mod(cA[k], cAp[k], cB[k], xa, p);
            rb = mul_add_mod(cA[k], cAp[k], cB[k], xb, p);
        }
        best[k] = FIRST ? min(ra, rb) : __vimin3_u32(best[k], ra, rb);
    }
}

template <int K, bool NARROW, bool FIRST>
__device__ __forceinline__ void walk1_random(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                             const uint32_t (&cAp)[K], const uint32_t (&cB)[K],
                                             uint32_t xa, uint32_t p) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        uint32_t ra = NARROW ? mul_add_mod_narrow(cA[k], cAp[k], cB[k], xa, p)
                             : mul_add_mod(cA[k], cAp[k], cB[k], xa, p);
        best[k] = FIRST ? ra : min(best[k], ra);
    }
}

// ---- asynchronous global->shared copies (cp.async / LDGSTS) ----
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(long long* dst, const int64_t* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

// Per-warp shared memory: a two-slot ring of item ids (the slot of the item being
// processed doubles as the slice-combine scratch once its rounds are done) and the
// CSR bounds of the current and next batch.
struct WarpSmem {
    uint32_t ids[2][kChunk];
    long long ip[2][kBatch + 2];
};

// Warp-uniform description of one work item.
struct ItemDesc {
    int64_t f0;    // first feature (index into ids)
    int64_t s;     // set index
    int32_t n;     // features in the item (0: skip / no item)
    int32_t sb;    // lane pass
    int32_t merge; // long set: merge with atomicMin, finalize later
};

__device__ __forceinline__ ItemDesc make_item(int64_t s, int sb, int64_t f0, int64_t hi, bool long_set) {
    ItemDesc d;
    const int64_t n = hi - f0;
    d.f0 = f0;
    d.s = s;
    d.sb = sb;
    d.n = n <= 0 ? 0 : (n > kChunk ? kChunk : (int32_t)n);
    d.merge = long_set;
    return d;
}

__device__ __forceinline__ ItemDesc no_item() {
    ItemDesc d;
    d.f0 = 0; d.s = 0; d.n = 0; d.sb = 0; d.merge = 0;
    return d;
}

// Stage an item's ids into a ring slot: lane-strided 4-byte async copies.
__device__ __forceinline__ void stage_ids(const SignArgs& A, const ItemDesc& d, uint32_t* slot, int lane) {
    const uint32_t* src = A.ids + d.f0;
    for (int o = lane; o < d.n; o += 32) cp_async4(slot + o, src + o);
}

// Batch b covers primary items [b*kBatch, b*kBatch + kBatch).  Their sets span
// [s_first, s_first + cnt); stage indptr[s_first .. s_first + cnt] (cnt+1 values).
__device__ __forceinline__ int64_t batch_first_set(const SignArgs& A, unsigned long long b) {
    const unsigned long long item = b * kBatch;
    return A.n_super == 1 ? (int64_t)item : (int64_t)(item / (unsigned)A.n_super);
}

__device__ __forceinline__ void stage_bounds(const SignArgs& A, unsigned long long b, unsigned long long n_batches,
                                             long long* ip, int lane) {
    if (b >= n_batches) return;
    const int64_t s0 = batch_first_set(A, b);
    const unsigned long long last_item = min(b * kBatch + kBatch, (unsigned long long)A.n_sets * A.n_super) - 1;
    const int64_t s1 = A.n_super == 1 ? (int64_t)last_item : (int64_t)(last_item / (unsigned)A.n_super);
    const int cnt = (int)(s1 - s0) + 2;  // indptr values needed
    if (lane < cnt) cp_async8(ip + lane, A.indptr + s0 + lane);
}

__device__ __forceinline__ ItemDesc batch_item(const SignArgs& A, unsigned long long b, int j, const long long* ip) {
    const unsigned long long item = b * kBatch + j;
    int64_t s;
    int sb = 0;
    if (A.n_super == 1) {
        s = (int64_t)item;
    } else {
        s = (int64_t)(item / (unsigned)A.n_super);
        sb = (int)(item - (unsigned long long)s * A.n_super);
    }
    const int64_t k = s - batch_first_set(A, b);
    const int64_t lo = ip[k], hi = ip[k + 1];
    return make_item(s, sb, lo, hi, (hi - lo) > kChunk);
}

// Per-thread hashing state: iterative start constants, or the K random-family lane constants.
template <int K, bool ITER>
struct LaneState {
    uint32_t tA, tAp, tB;
    uint32_t cA[ITER ? 1 : K], cAp[ITER ? 1 : K], cB[ITER ? 1 : K];
};

template <int K, bool ITER, bool NARROW, bool FIRST>
__device__ __forceinline__ void round2(uint32_t (&best)[K], const LaneState<K, ITER>& ls, uint32_t xa, uint32_t xb,
                                       uint32_t p, uint32_t bpar) {
    if constexpr (ITER) {
        const uint32_t ha = mul_add_mod(ls.tA, ls.tAp, ls.tB, xa, p);
        const uint32_t hb = mul_add_mod(ls.tA, ls.tAp, ls.tB, xb, p);
        walk2_iter<K, FIRST>(best, ha, reduce_once(xa + bpar, p), hb, reduce_once(xb + bpar, p), p);
    } else {
        walk2_random<K, NARROW, FIRST>(best, ls.cA, ls.cAp, ls.cB, xa, xb, p);
    }
}

template <int K, bool ITER, bool NARROW, bool FIRST>
__device__ __forceinline__ void round1(uint32_t (&best)[K], const LaneState<K, ITER>& ls, uint32_t xa,
                                       uint32_t p, uint32_t bpar) {
    if constexpr (ITER) {
        const uint32_t ha = mul_add_mod(ls.tA, ls.tAp, ls.tB, xa, p);
        walk1_iter<K, FIRST>(best, ha, reduce_once(xa + bpar, p), p);
    } else {
        walk1_random<K, NARROW, FIRST>(best, ls.cA, ls.cAp, ls.cB, xa, p);
    }
}

template <int K, bool ITER, bool NARROW, bool FIRST>
__device__ __forceinline__ void last_round(uint32_t (&best)[K], const LaneState<K, ITER>& ls, bool single,
                                           uint32_t xa, uint32_t xb, uint32_t p, uint32_t bpar, uint32_t& maxid) {
    if (single) {
        maxid = max(maxid, xa);
        round1<K, ITER, NARROW, FIRST>(best, ls, xa, p, bpar);
    } else {
        maxid = __vimax3_u32(maxid, xa, xb);
        round2<K, ITER, NARROW, FIRST>(best, ls, xa, xb, p, bpar);
    }
}

// Stage KP of each thread's minima (lanes k0..k0+KP) into the warp scratch `red`
// with a 16-byte-chunk XOR swizzle (conflict-free writes and reads).
template <int K, int K0>
__device__ __forceinline__ void store_slice(const uint32_t (&best)[K], uint32_t* red, int lane) {
    constexpr int KP = K < 32 ? K : 32;
    constexpr int NQ = KP / 4;
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int qq = q ^ (lane & SWZ);
        *reinterpret_cast<uint4*>(red + lane * KP + qq * 4) =
            make_uint4(best[K0 + 4 * q], best[K0 + 4 * q + 1], best[K0 + 4 * q + 2], best[K0 + 4 * q + 3]);
    }
}

// Combine the F slices for lanes k0..k0+KP of every lane group, recover the argmin
// ids and store them (or atomicMin the min hashes of a long set).
template <int K, typename OutT>
__device__ __forceinline__ void combine_emit(const SignArgs& A, const ItemDesc& cur, int k0, const uint32_t* red,
                                             const InvTab* epi_s, bool epi_smem, int lane, int F) {
    constexpr int KP = K < 32 ? K : 32;
    constexpr int NQ = KP / 4;
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;
    const uint32_t p = A.p;
    const int32_t N = A.n_hash;
    const int G = 32 / F;
    const int n_chunks = G * KP / 4;
    const bool vec_ok = ((N & 3) == 0);
    OutT* row = reinterpret_cast<OutT*>(A.out) + cur.s * (int64_t)N;
    for (int c = lane; c < n_chunks; c += 32) {
        const int l4 = 4 * c;
        const int gg = l4 / KP;
        const int kk = l4 - gg * KP;
        const int qk = kk / 4;
        const uint32_t* src = red + gg * F * KP;
        uint4 m = *reinterpret_cast<const uint4*>(src + (qk ^ ((gg * F) & SWZ)) * 4);
        int ff = 1;
        for (; ff + 1 < F; ff += 2) {
            const int w0 = gg * F + ff, w1 = w0 + 1;
            const uint4 v0 = *reinterpret_cast<const uint4*>(src + ff * KP + (qk ^ (w0 & SWZ)) * 4);
            const uint4 v1 = *reinterpret_cast<const uint4*>(src + (ff + 1) * KP + (qk ^ (w1 & SWZ)) * 4);
            m.x = __vimin3_u32(m.x, v0.x, v1.x); m.y = __vimin3_u32(m.y, v0.y, v1.y);
            m.z = __vimin3_u32(m.z, v0.z, v1.z); m.w = __vimin3_u32(m.w, v0.w, v1.w);
        }
        if (ff < F) {
            const int w0 = gg * F + ff;
            const uint4 v0 = *reinterpret_cast<const uint4*>(src + ff * KP + (qk ^ (w0 & SWZ)) * 4);
            m.x = min(m.x, v0.x); m.y = min(m.y, v0.y); m.z = min(m.z, v0.z); m.w = min(m.w, v0.w);
        }
        const int64_t i = (int64_t)cur.sb * A.L + (int64_t)gg * K + k0 + kk;
        if (cur.merge) {
            if (i + 0 < N) atomic_min_out(row + i + 0, m.x);
            if (i + 1 < N) atomic_min_out(row + i + 1, m.y);
            if (i + 2 < N) atomic_min_out(row + i + 2, m.z);
            if (i + 3 < N) atomic_min_out(row + i + 3, m.w);
            continue;
        }
        uint32_t x[4];
        const uint32_t h[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            InvTab t;
            if (epi_smem) {
                t = epi_s[i + e];
            } else {
                t = A.inv[min(i + e, (int64_t)A.n_tot - 1)];
            }
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

// One work item whose ids are staged in `slot`: rounds (the first initialises the
// minima; a last round with <= F features walks one feature per slice), then the
// slice combine in `slot` (the ids are consumed by then) and the epilogue.
template <int K, bool ITER, bool NARROW, typename OutT>
__device__ __forceinline__ void run_item(const SignArgs& A, const ItemDesc& cur, uint32_t* slot,
                                         LaneState<K, ITER>& ls, int& cur_sb, uint32_t& maxid,
                                         const InvTab* epi_s, bool epi_smem, int lane, int g, int f, int F) {
    const uint32_t p = A.p;
    const uint32_t bpar = A.b;
    if (cur.sb != cur_sb) {  // lane constants change only with the lane pass
        const int64_t i0 = (int64_t)cur.sb * A.L + (int64_t)g * K;
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
        cur_sb = cur.sb;
    }

    // rounds of 2F features; F is a power of two
    uint32_t best[K];
    const int n = cur.n;
    const int last = n - 1;
    const int sh = A.log2F + 1;
    const int rounds = (n + (1 << sh) - 1) >> sh;
    const bool single = rounds > 1 && (n - ((rounds - 1) << sh)) <= F;
    {
        const uint32_t xa = slot[min(f, last)], xb = slot[min(F + f, last)];
        maxid = __vimax3_u32(maxid, xa, xb);
        round2<K, ITER, NARROW, true>(best, ls, xa, xb, p, bpar);
    }
    // middle rounds are always full: no clamping, no branches
    const int full_end = (rounds - 1) << sh;
    int o = 2 * F + f;
#pragma unroll 1
    for (; o < full_end; o += 2 * F) {
        const uint32_t xa = slot[o], xb = slot[o + F];
        maxid = __vimax3_u32(maxid, xa, xb);
        round2<K, ITER, NARROW, false>(best, ls, xa, xb, p, bpar);
    }
    if (rounds > 1) {
        const uint32_t xa = slot[min(o, last)], xb = slot[min(o + F, last)];
        if (single) {
            maxid = max(maxid, xa);
            round1<K, ITER, NARROW, false>(best, ls, xa, p, bpar);
        } else {
            maxid = __vimax3_u32(maxid, xa, xb);
            round2<K, ITER, NARROW, false>(best, ls, xa, xb, p, bpar);
        }
    }
    __syncwarp();  // every lane is done reading ids before the slot becomes scratch
    constexpr int KP = K < 32 ? K : 32;
    static_assert(K / KP <= 2, "at most two combine passes");
#pragma unroll 1
    for (int h = 0; h < K / KP; ++h) {
        if (h == 0) store_slice<K, 0>(best, slot, lane);
        else store_slice<K, (K > KP ? KP : 0)>(best, slot, lane);
        __syncwarp();
        combine_emit<K, OutT>(A, cur, h * KP, slot, epi_s, epi_smem, lane, F);
        __syncwarp();
    }
}

// Where the next work item comes from: first the extra chunks of long sets (one
// atomic each), then batches of kBatch consecutive primary items whose CSR bounds
// are staged in shared memory one batch ahead.
struct ItemSource {
    int phase;                   // 0 extras, 1 batches, 2 done
    int j, slot_b, in_batch;
    unsigned long long b_cur, b_nxt, b_nxt2;
};

__device__ __forceinline__ ItemDesc next_item(const SignArgs& A, ItemSource& src, WarpSmem* ws, int lane,
                                              unsigned long long n_extra, unsigned long long n_primary,
                                              unsigned long long n_batches) {
    if (src.phase == 0) {
        unsigned long long e = 0;
        if (lane == 0) e = atomicAdd(&A.sched->next_extra, 1ull);
        e = __shfl_sync(0xffffffffu, e, 0);
        if (e < n_extra) {
            const Extra x = A.extra[e];
            const int64_t lo = A.indptr[x.set], hi = A.indptr[x.set + 1];
            return make_item(x.set, x.sb, lo + (int64_t)x.chunk * kChunk, hi, true);
        }
        // enter the batch phase: claim three batches, stage two batches of bounds
        src.phase = 1;
        if (lane == 0) {
            src.b_cur = atomicAdd(&A.sched->next, 1ull);
            src.b_nxt = atomicAdd(&A.sched->next, 1ull);
            src.b_nxt2 = atomicAdd(&A.sched->next, 1ull);
        }
        src.b_cur = __shfl_sync(0xffffffffu, src.b_cur, 0);
        src.b_nxt = __shfl_sync(0xffffffffu, src.b_nxt, 0);
        if (src.b_cur >= n_batches) {
            src.phase = 2;
            return no_item();
        }
        src.slot_b = 0;
        stage_bounds(A, src.b_cur, n_batches, ws->ip[0], lane);
        stage_bounds(A, src.b_nxt, n_batches, ws->ip[1], lane);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        src.j = 0;
        src.in_batch = (int)min((unsigned long long)kBatch, n_primary - src.b_cur * kBatch);
        return batch_item(A, src.b_cur, 0, ws->ip[0]);
    }
    if (src.phase == 2) return no_item();
    if (++src.j == src.in_batch) {
        src.j = 0;
        src.b_cur = src.b_nxt;
        src.slot_b ^= 1;
        src.b_nxt = __shfl_sync(0xffffffffu, src.b_nxt2, 0);
        if (src.b_cur >= n_batches) {
            src.phase = 2;
            return no_item();
        }
        // The new current batch's bounds were staged a batch ago; make sure they landed.
        cp_async_wait<0>();
        __syncwarp();
        stage_bounds(A, src.b_nxt, n_batches, ws->ip[src.slot_b ^ 1], lane);
        if (lane == 0) src.b_nxt2 = atomicAdd(&A.sched->next, 1ull);
        src.in_batch = (int)min((unsigned long long)kBatch, n_primary - src.b_cur * kBatch);
    }
    return batch_item(A, src.b_cur, src.j, ws->ip[src.slot_b]);
}

template <int K, bool ITER, bool NARROW, typename OutT>
__global__ void __launch_bounds__(kBlock, ITER ? 2 : 1) sign_kernel(SignArgs A) {
    extern __shared__ uint4 smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw) + warp;
    InvTab* epi_s = reinterpret_cast<InvTab*>(reinterpret_cast<WarpSmem*>(smem_raw) + kBlock / 32);

    const int F = A.F;
    const int g = lane >> A.log2F;
    const int f = lane & (F - 1);

    // Stage the epilogue table (B_i, A_i^{-1}, companion) in shared memory.
    const bool epi_smem = A.n_tot <= kEpiSmemLanes;
    if (epi_smem) {
        for (int i = threadIdx.x; i < A.n_tot; i += blockDim.x) epi_s[i] = A.inv[i];
        __syncthreads();
    }

    LaneState<K, ITER> ls;
    int cur_sb = -1;
    uint32_t maxid = 0;

    const unsigned long long n_extra = *((volatile unsigned long long*)&A.sched->n_extra);
    const unsigned long long n_primary = (unsigned long long)A.n_sets * A.n_super;
    const unsigned long long n_batches = (n_primary + kBatch - 1) / kBatch;
    ItemSource src;
    src.phase = 0;
    src.j = src.slot_b = src.in_batch = 0;
    src.b_cur = src.b_nxt = src.b_nxt2 = 0;

    // Item pipeline: the next item's ids are staged (cp.async) while the current runs.
    int slot = 0;
    ItemDesc cur = next_item(A, src, ws, lane, n_extra, n_primary, n_batches);
    stage_ids(A, cur, ws->ids[0], lane);
    cp_async_commit();
    while (src.phase != 2 || cur.n > 0) {
        const ItemDesc nxt = next_item(A, src, ws, lane, n_extra, n_primary, n_batches);
        stage_ids(A, nxt, ws->ids[slot ^ 1], lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        if (cur.n > 0)
            run_item<K, ITER, NARROW, OutT>(A, cur, ws->ids[slot], ls, cur_sb, maxid, epi_s, epi_smem, lane, g, f, F);
        cur = nxt;
        slot ^= 1;
    }
    cp_async_wait<0>();
    if (__any_sync(0xffffffffu, maxid >= A.p) && lane == 0 && A.status) atomicOr(A.status, MHB_STATUS_ID_GE_PRIME);
}

// Long sets: rows hold min hash values after the main kernel; invert in place.
template <typename OutT>
__global__ void finalize_kernel(SignArgs A) {
    const unsigned long long n_big = *((volatile unsigned long long*)&A.sched->n_big);
    const unsigned long long total = n_big * (unsigned long long)A.L;
    OutT* out = reinterpret_cast<OutT*>(A.out);
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long e = t / (unsigned)A.L;
        const int l = (int)(t - e * A.L);
        const int64_t key = A.big[e];
        const int64_t s = key / A.n_super;
        const int sb = (int)(key - s * A.n_super);
        const int64_t i = (int64_t)sb * A.L + l;
        if (i < A.n_hash) {
            OutT* cell = out + s * (int64_t)A.n_hash + i;
            *cell = (OutT)invert_lane(A, i, (uint32_t)*cell);
        }
    }
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

using SignKernelFn = void (*)(SignArgs);

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

static SignKernelFn select_kernel(int kind, bool narrow, int out_dtype, int K) {
    const bool i64 = out_dtype == MHB_OUT_I64;
    if (kind == KIND_ITERATIVE) {
        return i64 ? pick_kernel<true, false, long long>(K) : pick_kernel<true, false, uint32_t>(K);
    }
    if (narrow) return i64 ? pick_kernel<false, true, long long>(K) : pick_kernel<false, true, uint32_t>(K);
    return i64 ? pick_kernel<false, false, long long>(K) : pick_kernel<false, false, uint32_t>(K);
}

// Occupancy (CTAs per SM) per (kernel, device, dynamic smem); computed once.  The
// dynamic-smem limit is raised to the device maximum the first time a kernel is seen.
static int blocks_per_sm(SignKernelFn fn, size_t smem, const DeviceInfo& dev) {
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
    if (!seen)
        cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dev.smem_optin);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kBlock, smem) != cudaSuccess)
        occ = 1;
    if (occ < 1) occ = 1;
    if (n_cache < 512) cache[n_cache++] = Entry{(const void*)fn, dev.device, smem, occ};
    return occ;
}

int launch_sign(int kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t nnz,
                uint64_t a, uint64_t b, const uint32_t* ra, const uint32_t* rb, uint64_t prime,
                int32_t n_hash, void* out, int32_t out_dtype, int32_t* status, void* workspace,
                size_t workspace_bytes, cudaStream_t st) {
    clear_error();
    if (n_sets < 0 || nnz < 0) return set_error(MHB_ERR_INVALID, "n_sets and nnz must be >= 0");
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function, got %d", n_hash);
    if (prime < 3 || !is_prime_u64(prime)) return set_error(MHB_ERR_INVALID, "modulus %llu is not prime",
                                                             (unsigned long long)prime);
    if (prime >= (1ull << 31))
        return set_error(MHB_ERR_UNSUPPORTED, "prime %llu >= 2^31 is outside the u32 kernels' range",
                         (unsigned long long)prime);
    if (out_dtype != MHB_OUT_U32 && out_dtype != MHB_OUT_I64)
        return set_error(MHB_ERR_INVALID, "unknown out_dtype %d", out_dtype);
    if (kind == KIND_ITERATIVE) {
        if (a < 1 || a >= prime || b >= prime)
            return set_error(MHB_ERR_INVALID, "need 1 <= a < p and 0 <= b < p");
        if (a + (uint64_t)n_hash >= prime)
            return set_error(MHB_ERR_INVALID,
                             "need a + size < prime to keep every member invertible; got a=%llu, size=%d, "
                             "prime=%llu", (unsigned long long)a, n_hash, (unsigned long long)prime);
    } else if (ra == nullptr || rb == nullptr) {
        return set_error(MHB_ERR_INVALID, "random family needs device arrays a and b");
    }
    if (n_sets > 0 && (indptr == nullptr || out == nullptr))
        return set_error(MHB_ERR_INVALID, "null indptr/out");
    if (nnz > 0 && ids == nullptr) return set_error(MHB_ERR_INVALID, "null ids");

    const WorkspaceLayout wl = workspace_layout(n_sets, nnz, n_hash);
    if (workspace == nullptr || workspace_bytes < wl.total)
        return set_error(MHB_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", wl.total,
                         workspace_bytes);

    const Geometry geo = choose_geometry(kind, n_hash);
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
    A.n_tot = geo.n_tot;
    A.kind = kind;
    A.tab = reinterpret_cast<LaneTab*>(ws + wl.tab);
    A.inv = reinterpret_cast<InvTab*>(ws + wl.inv);
    A.sched = reinterpret_cast<Sched*>(ws + wl.sched);
    A.big = reinterpret_cast<int64_t*>(ws + wl.big);
    A.extra = reinterpret_cast<Extra*>(ws + wl.extra);
    A.status = status;
    A.out = out;
    A.ra = ra;
    A.rb = rb;

    int rc = cuda_check(cudaMemsetAsync(A.sched, 0, sizeof(Sched), st), "memset sched");
    if (rc) return rc;
    if (status) {
        rc = cuda_check(cudaMemsetAsync(status, 0, sizeof(int32_t), st), "memset status");
        if (rc) return rc;
    }
    if (n_sets == 0) return MHB_OK;

    DeviceInfo dev;
    rc = current_device_info(&dev);
    if (rc) return rc;

    {
        int64_t work = n_sets > geo.n_tot ? n_sets : geo.n_tot;
        int64_t blocks = (work + 255) / 256;
        int64_t cap = (int64_t)dev.sms * 8;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        if (out_dtype == MHB_OUT_I64)
            setup_kernel<long long><<<(unsigned)blocks, 256, 0, st>>>(A);
        else
            setup_kernel<uint32_t><<<(unsigned)blocks, 256, 0, st>>>(A);
        rc = cuda_check(cudaGetLastError(), "setup_kernel launch");
        if (rc) return rc;
    }

    const bool narrow = (3ull * prime) < (1ull << 32);
    SignKernelFn fn = select_kernel(kind, narrow, out_dtype, geo.K);
    if (!fn) return set_error(MHB_ERR_INVALID, "no kernel instance for K=%d", geo.K);
    const size_t smem = (size_t)(kBlock / 32) * sizeof(WarpSmem) +
                        (geo.n_tot <= kEpiSmemLanes ? (size_t)geo.n_tot * sizeof(InvTab) : 0);
    const int occ = blocks_per_sm(fn, smem, dev);
    const int64_t items_ub = (n_sets * geo.n_super + kBatch - 1) / kBatch + (nnz / kChunk) * geo.n_super;
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
    fn<<<(unsigned)blocks, kBlock, smem, st>>>(A);
    if (prof_slot >= 0) cudaEventRecord(g_prof_ev[2 * prof_slot + 1], st);
    rc = cuda_check(cudaGetLastError(), "sign_kernel launch");
    if (rc) return rc;

    {
        int64_t fb = (int64_t)dev.sms * 2;
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

extern "C" int mhb_sign_random_csr(const int64_t* indptr, const uint32_t* ids, int64_t n_sets,
                                   int64_t nnz, const uint32_t* a, const uint32_t* b, uint64_t prime,
                                   int32_t n_hash, void* out, int32_t out_dtype, int32_t* status,
                                   void* workspace, size_t workspace_bytes, void* stream) {
    return mhb::launch_sign(mhb::KIND_RANDOM, indptr, ids, n_sets, nnz, 0, 0, a, b, prime, n_hash,
                            out, out_dtype, status, workspace, workspace_bytes,
                            static_cast<cudaStream_t>(stream));
}
