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
        v.inv = inv_mod(w, p);
        v.invp = shoup_companion(v.inv, p);
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

__device__ __forceinline__ uint32_t invert_lane(const SignArgs& A, int64_t i, uint32_t h) {
    // x = (h - B_i) * A_i^{-1} mod p
    const uint32_t p = A.p;
    const uint32_t B = __ldg(&A.tab[i].B);
    const InvTab v = A.inv[i];
    uint32_t d = h - B;
    d = __viaddmin_u32(d, p, d);  // d in [0,p)
    return reduce_once(shoup_lazy(v.inv, v.invp, d, p), p);
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

template <int K>
__device__ __forceinline__ void walk2_iter(uint32_t (&best)[K], uint32_t ha, uint32_t da,
                                           uint32_t hb, uint32_t db, uint32_t p) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        best[k] = __vimin3_u32(best[k], ha, hb);
        if (k + 1 < K) {
            ha = reduce_once(ha + da, p);
            hb = reduce_once(hb + db, p);
        }
    }
}

template <int K>
__device__ __forceinline__ void walk1_iter(uint32_t (&best)[K], uint32_t ha, uint32_t da, uint32_t p) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        best[k] = min(best[k], ha);
        if (k + 1 < K) ha = reduce_once(ha + da, p);
    }
}

template <int K, bool NARROW>
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
        best[k] = __vimin3_u32(best[k], ra, rb);
    }
}

template <int K, bool NARROW>
__device__ __forceinline__ void walk1_random(uint32_t (&best)[K], const uint32_t (&cA)[K],
                                             const uint32_t (&cAp)[K], const uint32_t (&cB)[K],
                                             uint32_t xa, uint32_t p) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        uint32_t ra = NARROW ? mul_add_mod_narrow(cA[k], cAp[k], cB[k], xa, p)
                             : mul_add_mod(cA[k], cAp[k], cB[k], xa, p);
        best[k] = min(best[k], ra);
    }
}

template <int K, bool ITER, bool NARROW, typename OutT>
__global__ void __launch_bounds__(kBlock) sign_kernel(SignArgs A) {
    extern __shared__ uint4 smem_raw[];
    constexpr int NQ = K / 4;                       // 16-byte chunks per thread
    constexpr int SWZ = (NQ < 8 ? NQ : 8) - 1;      // chunk swizzle mask
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* red = reinterpret_cast<uint32_t*>(smem_raw) + warp * 32 * K;

    const uint32_t p = A.p;
    const uint32_t bpar = A.b;
    const int F = A.F;
    const int g = lane >> A.log2F;
    const int f = lane & (F - 1);
    const int L = A.L;
    const int32_t N = A.n_hash;
    OutT* out = reinterpret_cast<OutT*>(A.out);

    const unsigned long long n_extra = *((volatile unsigned long long*)&A.sched->n_extra);
    const unsigned long long total = n_extra + (unsigned long long)A.n_sets * A.n_super;

    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(&A.sched->next, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);

    int cur_sb = -1;
    uint32_t cA[K], cAp[K], cB[K];
    bool bad = false;

    while (item < total) {
        unsigned long long nxt = 0;
        if (lane == 0) nxt = atomicAdd(&A.sched->next, 1ull);

        int64_t s, f0, f1;
        int sb;
        bool merge;
        if (item < n_extra) {
            const Extra e = A.extra[item];
            s = e.set;
            sb = e.sb;
            const int64_t lo = A.indptr[s], hi = A.indptr[s + 1];
            f0 = lo + (int64_t)e.chunk * kChunk;
            f1 = min(f0 + (int64_t)kChunk, hi);
            merge = true;
        } else {
            const unsigned long long pid = item - n_extra;
            if (A.n_super == 1) {
                s = (int64_t)pid;
                sb = 0;
            } else {
                s = (int64_t)(pid / (unsigned)A.n_super);
                sb = (int)(pid - (unsigned long long)s * A.n_super);
            }
            const int64_t lo = A.indptr[s], hi = A.indptr[s + 1];
            f0 = lo;
            f1 = min(lo + (int64_t)kChunk, hi);
            merge = (hi - lo) > kChunk;
        }

        if (f1 > f0) {
            const int64_t i0 = (int64_t)sb * L + (int64_t)g * K;
            uint32_t tA = 0, tAp = 0, tB = 0;
            if constexpr (ITER) {
                const LaneTab t = A.tab[i0];
                tA = t.A; tAp = t.Ap; tB = t.B;
            } else {
                if (sb != cur_sb) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const LaneTab t = A.tab[i0 + k];
                        cA[k] = t.A; cAp[k] = t.Ap; cB[k] = t.B;
                    }
                    cur_sb = sb;
                }
            }

            uint32_t best[K];
#pragma unroll
            for (int k = 0; k < K; ++k) best[k] = 0xffffffffu;

            const uint32_t* ids = A.ids;
            const int64_t n = f1 - f0;
            const int64_t step = 2 * (int64_t)F;
            const int64_t n_pair_rounds = n / step;
            const int64_t rem = n - n_pair_rounds * step;

            // ---- full rounds: every slice has two valid features ----
            if (n_pair_rounds > 0) {
                int64_t ja = f0 + f;
                uint32_t xa = __ldg(ids + ja), xb = __ldg(ids + ja + F);
                for (int64_t r = 0; r < n_pair_rounds; ++r) {
                    // prefetch next round (clamped to a valid address)
                    int64_t jn = ja + step;
                    const int64_t jna = jn < f1 ? jn : f0;
                    const int64_t jnb = jn + F < f1 ? jn + F : f0;
                    const uint32_t xa_n = __ldg(ids + jna), xb_n = __ldg(ids + jnb);
                    bad |= (xa >= p) | (xb >= p);
                    if constexpr (ITER) {
                        const uint32_t ha = mul_add_mod(tA, tAp, tB, xa, p);
                        const uint32_t hb = mul_add_mod(tA, tAp, tB, xb, p);
                        const uint32_t da = reduce_once(xa + bpar, p);
                        const uint32_t db = reduce_once(xb + bpar, p);
                        walk2_iter<K>(best, ha, da, hb, db, p);
                    } else {
                        walk2_random<K, NARROW>(best, cA, cAp, cB, xa, xb, p);
                    }
                    xa = xa_n;
                    xb = xb_n;
                    ja = jn;
                }
            }
            // ---- tail: rem < 2F features left ----
            if (rem > 0) {
                const int64_t base = f0 + n_pair_rounds * step;
                if (rem > F) {
                    const int64_t ja = base + f;            // always < f1 since f < F < rem
                    const int64_t jb = base + F + f;
                    const uint32_t xa = __ldg(ids + ja);
                    const uint32_t xb = __ldg(ids + (jb < f1 ? jb : ja));
                    bad |= (xa >= p) | (xb >= p);
                    if constexpr (ITER) {
                        const uint32_t ha = mul_add_mod(tA, tAp, tB, xa, p);
                        const uint32_t hb = mul_add_mod(tA, tAp, tB, xb, p);
                        const uint32_t da = reduce_once(xa + bpar, p);
                        const uint32_t db = reduce_once(xb + bpar, p);
                        walk2_iter<K>(best, ha, da, hb, db, p);
                    } else {
                        walk2_random<K, NARROW>(best, cA, cAp, cB, xa, xb, p);
                    }
                } else {
                    const int64_t ja = base + f;
                    const uint32_t xa = __ldg(ids + (ja < f1 ? ja : base));
                    bad |= (xa >= p);
                    if constexpr (ITER) {
                        const uint32_t ha = mul_add_mod(tA, tAp, tB, xa, p);
                        const uint32_t da = reduce_once(xa + bpar, p);
                        walk1_iter<K>(best, ha, da, p);
                    } else {
                        walk1_random<K, NARROW>(best, cA, cAp, cB, xa, p);
                    }
                }
            }

            // ---- combine the F slices through the warp's smem tile ----
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int qq = q ^ (lane & SWZ);
                *reinterpret_cast<uint4*>(red + lane * K + qq * 4) =
                    make_uint4(best[4 * q], best[4 * q + 1], best[4 * q + 2], best[4 * q + 3]);
            }
            __syncwarp();
            const int n_chunks = L / 4;
            const bool vec_ok = ((N & 3) == 0);
            OutT* row = out + s * (int64_t)N;
            for (int c = lane; c < n_chunks; c += 32) {
                const int l = 4 * c;
                const int gg = l / K;
                const int qk = (l % K) / 4;
                uint4 m = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                for (int ff = 0; ff < F; ++ff) {
                    const int w = gg * F + ff;
                    const int qq = qk ^ (w & SWZ);
                    const uint4 v = *reinterpret_cast<const uint4*>(red + w * K + qq * 4);
                    m.x = min(m.x, v.x); m.y = min(m.y, v.y);
                    m.z = min(m.z, v.z); m.w = min(m.w, v.w);
                }
                const int64_t i = (int64_t)sb * L + l;
                if (merge) {
                    if (i + 0 < N) atomic_min_out(row + i + 0, m.x);
                    if (i + 1 < N) atomic_min_out(row + i + 1, m.y);
                    if (i + 2 < N) atomic_min_out(row + i + 2, m.z);
                    if (i + 3 < N) atomic_min_out(row + i + 3, m.w);
                } else if (vec_ok && i + 3 < N) {
                    store4(row + i, invert_lane(A, i, m.x), invert_lane(A, i + 1, m.y),
                           invert_lane(A, i + 2, m.z), invert_lane(A, i + 3, m.w));
                } else {
                    if (i + 0 < N) row[i + 0] = (OutT)invert_lane(A, i + 0, m.x);
                    if (i + 1 < N) row[i + 1] = (OutT)invert_lane(A, i + 1, m.y);
                    if (i + 2 < N) row[i + 2] = (OutT)invert_lane(A, i + 2, m.z);
                    if (i + 3 < N) row[i + 3] = (OutT)invert_lane(A, i + 3, m.w);
                }
            }
            __syncwarp();
        }
        item = __shfl_sync(0xffffffffu, nxt, 0);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && A.status) atomicOr(A.status, MHB_STATUS_ID_GE_PRIME);
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

// Occupancy (CTAs per SM) per kernel function; computed once per device.
static int blocks_per_sm(SignKernelFn fn, size_t smem, int device) {
    static std::mutex mu;
    struct Entry { const void* fn; int dev; int occ; };
    static Entry cache[256];
    static int n_cache = 0;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n_cache; ++i)
        if (cache[i].fn == (const void*)fn && cache[i].dev == device) return cache[i].occ;
    cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kBlock, smem) != cudaSuccess)
        occ = 1;
    if (occ < 1) occ = 1;
    if (n_cache < 256) cache[n_cache++] = Entry{(const void*)fn, device, occ};
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
    const size_t smem = (size_t)(kBlock / 32) * 32 * geo.K * sizeof(uint32_t);
    const int occ = blocks_per_sm(fn, smem, dev.device);
    const int64_t items_ub = n_sets * geo.n_super + (nnz / kChunk) * geo.n_super;
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
