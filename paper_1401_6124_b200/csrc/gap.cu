// gap.cu -- output-sensitive signing for the iterative family (kernels.py:44-73).
//
// The iterative generator makes lane i's hash of a feature an arithmetic progression
// mod p:  h_i(x) = ((a+i) x + i b) mod p = (h_0(x) + i d) mod p,  d = (x + b) mod p
// (families.py:124-131, kernels.py:62-72).  A signature entry is min_x h_i(x), and with n
// features that minimum is almost surely below T = p c / n.  So instead of VISITING every
// (feature, lane) pair -- N n visits per set, what sign_kernel does at 2.66 instructions
// each -- this kernel ENUMERATES, per feature, only the lanes i < N with h_i(x) < T: about
// N c / n of them, N c per set whatever its size.
//
// Enumeration (three-gap / Slater structure of a rotation, all in exact integers).  For an
// interval [0, L) the first-return map of v -> v + d mod p is a two-interval exchange
//     v <  w : v += u, i += n          (u = n d mod p,  the smallest "upward" return)
//     v >= w : v -= w, i += m          (w = -m d mod p, the smallest "downward" return)
// with L = u + w.  It starts as the rotation itself (u = d, w = p - d, n = m = 1, L = p)
// and shrinks Euclid-style: u >= w lets L drop by j w (u -= j w, n += j m), else by j u
// (w -= j u, m += j n); the orbit's first entry point (v, i) is carried along with at most
// one jump per level.  The descent stops at the last level with L >= T, where u, w < T,
// and the return map of [0, T) itself has three branches (Slater):
//     v <  T - u : (+u, +n)      v >= w : (-w, +m)      else : (u - w, n + m).
// Each hit is one `red.shared.min` into the set's N running minima in shared memory.
//
// Exactness.  Every recorded value is a true hash value, and every h_i(x) < T is recorded;
// so an entry whose minimum ends below T is the exact minimum.  The others (probability
// ~e^-c each) are recomputed from all the set's features (fallback list, a thread per
// entry).  c = ln(n) balances the two costs (ln(0.4 n) .. ln(1.5 n) swept on cfg4).  The
// argmin id is recovered from the minimum hash as in sign_kernel: x = (h - B_i) A_i^-1
// mod p.  The threshold decides cost only, never the result: a set of n copies of one id
// sends nearly every lane to the fallback (about 3x the visiting kernel's time for that
// set) and is still signed exactly.
//
// Work per tile of G consecutive sets (one CTA, G N minima in shared memory): thread k
// takes features k, k + 256, ... of the tile's contiguous id range; then the CTA inverts
// and stores the G rows with 16-byte stores, resets the minima it read and lists the
// entries for the fallback.  tests/test_gap_enumeration.py restates the descent in Python
// against brute force; tests/test_gpu_gap.py and tools/stress_gap.py pin the kernel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.h"
#include "modarith.cuh"
#include "sign_internal.h"

namespace mhb {

namespace {

constexpr int kGapThreads = 256;  // default CTA size (template parameter THREADS)
constexpr int kGapMaxSets = 64;        // sets per tile (upper bound)
constexpr int kGapFailCap = 512;       // fallback list entries per tile, two lists (overflow: marked minima)
constexpr size_t kGapBestBytes = 104 * 1024;  // running minima per CTA: two CTAs per SM at most

struct GapArgs {
    const int64_t* indptr;
    const uint32_t* ids;
    int64_t n_sets;
    uint32_t p, b, a, ap;   // a mod p and its Shoup companion: h_0(x) = a x mod p
    int32_t n_hash;
    int32_t G;              // sets per tile
    float cmul;             // threshold scale inside the log (1: measured best on cfg4, 0.4-1.5 swept)
    uint32_t one;           // 1, opaque to the compiler (IMAD-spelled adds)
    const LaneTab* tab;
    const InvTab* inv;
    unsigned long long* next;  // tile counter (zeroed by the caller)
    int32_t* status;
    void* out;
};

__device__ __forceinline__ void reds_min(uint32_t saddr, uint32_t v) {
    asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

__device__ __forceinline__ void gap_store4(uint32_t* dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(a, b, c, d);
}
__device__ __forceinline__ void gap_store4(long long* dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    longlong2* v = reinterpret_cast<longlong2*>(dst);
    v[0] = make_longlong2((long long)a, (long long)b);
    v[1] = make_longlong2((long long)c, (long long)d);
}

__device__ __forceinline__ uint32_t gap_invert(const InvTab& t, uint32_t h, uint32_t p) {
    uint32_t d = h - t.B;
    d = __viaddmin_u32(d, p, d);
    return reduce_once(shoup_lazy(t.inv, t.invp, d, p), p);
}

// All lanes i < N with h_i(x) < T for one feature: descent, then the three-branch walk.
// `sbase` is the shared address of the set's minima row.
__device__ __forceinline__ void enumerate_feature(uint32_t x, uint32_t T, uint32_t sbase, const GapArgs& A) {
    const uint32_t p = A.p, N = (uint32_t)A.n_hash;
    const uint32_t d = reduce_once(x + A.b, p);
    uint32_t v = reduce_once(shoup_lazy(A.a, A.ap, x, p), p);  // h_0(x)
    uint32_t t = 0;
    uint32_t u, n, w, m;
    if (d == 0) {
        // constant orbit: every lane hashes x to h_0(x)
        if (v >= T) return;
        u = 0; n = 1; w = T; m = N;
    } else {
        u = d; n = 1; w = p - d; m = 1;
        uint32_t L = p;
        for (;;) {
            const uint32_t mn = min(u, w);
            if (mn == 0 || L - mn < T || t >= N) break;
            // One level, both cases in one instruction stream (a warp's lanes differ in
            // which return is the larger): the larger return `big` (time tb) loses j
            // copies of the smaller `mn` (time ts), and so does L.
            const bool up_big = u >= w;  // reduce u by w, else w by u
            const uint32_t big = up_big ? u : w, tb = up_big ? n : m, ts = up_big ? m : n;
            const uint32_t j = min(big, L - T) / mn;
            const uint32_t L2 = L - j * mn;
            // the entry point, if it lies in the part cut off [L2, L): up_big: s = q + 1
            // downward steps of w; else the one downward step of the level it sits in,
            // w - q u (time m + q n)
            const uint32_t q = (up_big ? v - L2 : L - 1u - v) / mn;
            const uint32_t dv = up_big ? (q + 1u) * mn : big - q * mn;
            const uint32_t dt = up_big ? (q + 1u) * ts : tb + q * ts;
            if (v >= L2) {
                v -= dv;
                t += dt;
            }
            const uint32_t big2 = big - j * mn, tb2 = tb + j * ts;
            if (up_big) {
                u = big2;
                n = tb2;
            } else {
                w = big2;
                m = tb2;
            }
            L = L2;
        }
        if (t >= N) return;
        if (v >= T) {  // the level's interval is [0, L) with T <= L: one more return step
            v -= w;
            t += m;
            if (t >= N) return;
        }
    }
    // return map of [0, T): the upward step when v < w, then the downward step unless that
    // landed inside [0, T) (the third branch is both); steps in bytes of the minima row,
    // clipped to the row
    const uint32_t n4 = min(n, N) * 4u, m4 = min(m, N) * 4u;
    const uint32_t negw = 0u - w;
    uint32_t addr = sbase + t * 4u;
    const uint32_t end = sbase + N * 4u;
    // The selects are predicated adds: the value's on the FMA pipe (multiply by an opaque
    // one), the address's on the ALU pipe, so neither pipe carries all nine operations.
    const uint32_t one = A.one;
    while (addr < end) {
        reds_min(addr, v);
        asm volatile(
            "{\n\t"
            // up: the upward step; stay: it landed inside [0, T).  Every other case (no
            // upward step, or one that overshot T) takes the downward step, so the three
            // branches are two predicated pairs.
            ".reg .pred up, stay;\n\t"
            "setp.lt.u32 up, %0, %2;\n\t"
            "@up  mad.lo.u32 %0, %3, %8, %0;\n\t"
            "@up  add.u32 %1, %1, %5;\n\t"
            "setp.lt.and.u32 stay, %0, %7, up;\n\t"
            "@!stay mad.lo.u32 %0, %4, %8, %0;\n\t"
            "@!stay add.u32 %1, %1, %6;\n\t"
            "}"
            : "+r"(v), "+r"(addr)
            : "r"(w), "r"(u), "r"(negw), "r"(n4), "r"(m4), "r"(T), "r"(one));
    }
}

// Entry (set s, lane i) whose minimum stayed >= T: the exact minimum over every feature.
template <typename OutT>
__device__ __forceinline__ void fallback_entry(const GapArgs& A, int64_t f0, int64_t f1, uint32_t i, OutT* row) {
    const uint32_t p = A.p;
    const LaneTab lt = A.tab[i];
    uint32_t h = 0xFFFFFFFFu;
    for (int64_t f = f0; f < f1; ++f) h = min(h, mul_add_mod(lt.A, lt.Ap, lt.B, __ldg(A.ids + f), p));
    row[i] = (OutT)gap_invert(A.inv[i], h, p);
}

// The entries of one lane quad whose minimum stayed at or above the threshold: one
// counter bump per thread, then the list; the list full, the entry's (already reset)
// minimum is marked instead and the tile makes one more pass over its minima.
constexpr uint32_t kGapRedo = 0xFFFFFFFEu;
__device__ __forceinline__ void push_failures(uint32_t mask, uint32_t e0, uint32_t* best, unsigned* fcount,
                                              uint32_t* flist) {
    // PTX atom: the C++ atomicAdd here compiles to a warp-wide scan (five shuffles) that
    // every warp with one failing lane would run
    unsigned slot;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                 : "=r"(slot)
                 : "r"((uint32_t)__cvta_generic_to_shared(fcount)), "r"((unsigned)__popc(mask))
                 : "memory");
    // one trip per failing entry (almost always one): four unrolled tests cost every
    // warp with a failing lane ~30 instructions at two or three lanes
#pragma unroll 1
    for (; mask; mask &= mask - 1u, ++slot) {
        const uint32_t e = e0 + (uint32_t)__ffs((int)mask) - 1u;
        if (slot < kGapFailCap) flist[slot] = e;
        else best[e] = kGapRedo;
    }
}

// INV != 0: n_hash is a multiple of 4 up to 2048, and this thread's (at most two) lane quads'
// argmin-recovery constants are in registers for the row pass: INV = 1 for the whole launch
// (few sets per tile, cfg4: 17.9 against 18.7 ms), INV = 2 reloaded per tile just before the
// barrier, which frees 24 registers in the feature phase (many sets per tile, cfg3: 3.50
// against 3.70 ms).
template <typename OutT, int INV, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS == 256 ? 4 : 1) sign_gap_kernel(GapArgs A) {
    extern __shared__ uint4 gap_smem4[];
    // offsets and fallback list of the current and of the previous tile: a tile's fallback
    // entries are recomputed during the NEXT tile's feature phase (no phase of its own, no
    // barrier after it, and its uneven per-thread work averages into the longer phase)
    __shared__ long long sip2[2][kGapMaxSets + 1];
    __shared__ uint32_t sT[kGapMaxSets];
    __shared__ uint32_t flist2[2][kGapFailCap];
    __shared__ unsigned fcount2[2];
    __shared__ unsigned fnext2[2];   // the lists' claim cursors
    __shared__ unsigned long long s_tile[2];
    uint32_t* best = reinterpret_cast<uint32_t*>(gap_smem4);
    const uint32_t sbest = (uint32_t)__cvta_generic_to_shared(best);
    const int tid = threadIdx.x;
    const uint32_t p = A.p, N = (uint32_t)A.n_hash;
    const int64_t n_tiles = (A.n_sets + A.G - 1) / A.G;
    bool bad_id = false;
    constexpr bool REG_INV = INV != 0;
    InvTab rinv[REG_INV ? 8 : 1];
    auto load_inv = [&]() {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t i = ((uint32_t)tid + (uint32_t)(k / 4) * THREADS) * 4u + (uint32_t)(k & 3);
            const uint4 tv = __ldg(reinterpret_cast<const uint4*>(A.inv) + min(i, N - 1u));
            rinv[k].B = tv.x; rinv[k].inv = tv.y; rinv[k].invp = tv.z; rinv[k].pad = tv.w;
        }
    };
    if (INV == 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t i = ((uint32_t)tid + (uint32_t)(k / 4) * THREADS) * 4u + (uint32_t)(k & 3);
            rinv[k] = A.inv[min(i, N - 1u)];
        }
    }

    // minima start at UINT_MAX; the row pass below resets what it reads
    for (uint32_t q = tid; q < (uint32_t)A.G * N / 4u + 1u; q += THREADS)
        gap_smem4[q] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (tid == 0) s_tile[0] = atomicAdd(A.next, 1ull);
    if (tid < 2) fcount2[tid] = fnext2[tid] = 0;
    int64_t g0_prev = 0;
    int Gt_prev = 0;
    // the previous tile's fallback entries (list, then -- list overflow -- the marked minima)
    auto previous_fallbacks = [&](int prv, bool marked_only) {
        OutT* outp = reinterpret_cast<OutT*>(A.out) + g0_prev * (int64_t)N;
        const long long* sp = sip2[prv];
        const unsigned nfail = fcount2[prv];
        if (marked_only) {
            if (nfail > kGapFailCap) {
                const uint32_t ents = (uint32_t)Gt_prev * N;
                for (uint32_t e = tid; e < ents; e += THREADS)
                    if (best[e] == kGapRedo) {
                        best[e] = 0xFFFFFFFFu;
                        const uint32_t s = e / N, i = e - s * N;
                        fallback_entry<OutT>(A, sp[s], sp[s + 1], i, outp + (int64_t)s * N);
                    }
                __syncthreads();  // the minima are clean before the next feature phase
            }
            return;
        }
        // warps claim the list 32 entries at a time, AFTER their features: the warps that
        // finish the feature phase early take the entries instead of waiting at the barrier
        const unsigned nf = min(nfail, (unsigned)kGapFailCap);
        for (;;) {
            unsigned base = 0;
            if ((tid & 31) == 0) base = atomicAdd(&fnext2[prv], 32u);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base >= nf) break;
            const unsigned k = base + (unsigned)(tid & 31);
            if (k < nf) {
                const uint32_t e = flist2[prv][k], s = e / N, i = e - s * N;
                fallback_entry<OutT>(A, sp[s], sp[s + 1], i, outp + (int64_t)s * N);
            }
        }
    };
    int par = 0;
    for (;; par ^= 1) {
        __syncthreads();  // the tile before last's shared state is no longer read; s_tile[par] is set
        const int64_t tile = (int64_t)s_tile[par];
        if (tile >= n_tiles) break;
        long long* sip = sip2[par];
        uint32_t* flist = flist2[par];
        unsigned& fcount = fcount2[par];
        if (tid == 0) {
            s_tile[par ^ 1] = atomicAdd(A.next, 1ull);  // the next tile, claimed a tile ahead
            fcount = 0;
            fnext2[par] = 0;
        }
        const int64_t g0 = tile * A.G;
        const int Gt = (int)min((long long)A.G, (long long)(A.n_sets - g0));
        if (tid <= Gt) {
            const long long i0 = A.indptr[g0 + tid];
            sip[tid] = i0;
            if (tid < Gt) {
                // T = p c / n with c = ln(cmul n) >= 1: entries miss it with probability ~e^-c
                const long long n = A.indptr[g0 + tid + 1] - i0;
                uint32_t T = 0;
                if (n > 0) {
                    const float nf = (float)n;
                    const float c = fmaxf(1.0f, __logf(A.cmul * nf));
                    const float Tf = (float)p * (c / nf);
                    T = Tf >= (float)p ? p : max(1u, (uint32_t)Tf);
                }
                sT[tid] = T;
            }
        }
        __syncthreads();
        previous_fallbacks(par ^ 1, true);
        const int64_t fbeg = sip[0], fend = sip[Gt];
        for (int64_t f = fbeg + tid; f < fend; f += THREADS) {
            int lo = 0, hi = Gt;  // the set holding feature f: largest s with sip[s] <= f
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (sip[mid] <= f) lo = mid; else hi = mid;
            }
            const uint32_t x = __ldg(A.ids + f);
            if (x >= p) {
                bad_id = true;
                continue;
            }
            enumerate_feature(x, sT[lo], sbest + (uint32_t)lo * N * 4u, A);
        }
        previous_fallbacks(par ^ 1, false);
        if (INV == 2) load_inv();  // lands during the barrier
        __syncthreads();
        // rows out: minima below T are exact; the rest go to the fallback list
        OutT* out = reinterpret_cast<OutT*>(A.out) + g0 * (int64_t)N;
        if ((N & 3u) == 0) {
            const uint32_t nq = N / 4u;
            for (int s = 0; s < Gt; ++s) {
                const uint32_t T = sT[s];
                OutT* row = out + (int64_t)s * N;
                uint4* hrow = gap_smem4 + (uint32_t)s * nq;
                if (REG_INV) {
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const uint32_t q = tid + r * THREADS;
                        if (q < nq) {
                            const uint4 h4 = hrow[q];
                            hrow[q] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
                            const uint32_t hs[4] = {h4.x, h4.y, h4.z, h4.w};
                            uint32_t x[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) x[k] = gap_invert(rinv[r * 4 + k], hs[k], p);
                            gap_store4(row + q * 4u, x[0], x[1], x[2], x[3]);
                            if (max(max(hs[0], hs[1]), max(hs[2], hs[3])) >= T) {
                                const uint32_t mask = (hs[0] >= T ? 1u : 0u) | (hs[1] >= T ? 2u : 0u) |
                                                      (hs[2] >= T ? 4u : 0u) | (hs[3] >= T ? 8u : 0u);
                                push_failures(mask, (uint32_t)s * N + q * 4u, best, &fcount, flist);
                            }
                        }
                    }
                } else {
                    const uint4* inv4 = reinterpret_cast<const uint4*>(A.inv);
                    for (uint32_t q = tid; q < nq; q += THREADS) {
                        const uint4 h4 = hrow[q];
                        hrow[q] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
                        const uint32_t hs[4] = {h4.x, h4.y, h4.z, h4.w};
                        uint32_t x[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint4 tv = __ldg(inv4 + q * 4u + k);
                            InvTab it;
                            it.B = tv.x; it.inv = tv.y; it.invp = tv.z; it.pad = tv.w;
                            x[k] = gap_invert(it, hs[k], p);
                        }
                        gap_store4(row + q * 4u, x[0], x[1], x[2], x[3]);
                        if (max(max(hs[0], hs[1]), max(hs[2], hs[3])) >= T) {
                            const uint32_t mask = (hs[0] >= T ? 1u : 0u) | (hs[1] >= T ? 2u : 0u) |
                                                  (hs[2] >= T ? 4u : 0u) | (hs[3] >= T ? 8u : 0u);
                            push_failures(mask, (uint32_t)s * N + q * 4u, best, &fcount, flist);
                        }
                    }
                }
            }
        } else {
            const uint32_t ents = (uint32_t)Gt * N;
            for (uint32_t e = tid; e < ents; e += THREADS) {
                const uint32_t s = e / N, i = e - s * N;
                const uint32_t h = best[e];
                best[e] = 0xFFFFFFFFu;
                out[e] = (OutT)gap_invert(A.inv[i], h, p);
                if (h >= sT[s]) {
                    const unsigned slot = atomicAdd(&fcount, 1u);
                    if (slot < kGapFailCap) flist[slot] = e;
                    else best[e] = kGapRedo;
                }
            }
        }
        g0_prev = g0;
        Gt_prev = Gt;
    }
    // the last tile's fallback entries (every thread is past the barrier that followed its row pass)
    previous_fallbacks(par ^ 1, true);
    previous_fallbacks(par ^ 1, false);
    if (bad_id && A.status) atomicOr(A.status, MHB_STATUS_ID_GE_PRIME);
}

}  // namespace

int gap_sets_per_tile(int32_t n_hash) {
    const int64_t g = (int64_t)kGapBestBytes / ((int64_t)n_hash * 4);
    return (int)std::min<int64_t>(g, kGapMaxSets);
}

// Sets per tile for a batch: the tile's features are dealt to the CTA's threads in
// rounds, so pick the count whose expected features (plus one sigma, Poisson-like) waste
// the least of the last round.
static int gap_pick_sets(int32_t n_hash, int64_t n_sets, int64_t nnz, int threads) {
    const int gmax = gap_sets_per_tile(n_hash);
    const double mean = std::max(1.0, (double)nnz / (double)std::max<int64_t>(n_sets, 1));
    int best = 1;
    double best_eff = 0.0;
    // four resident CTAs (~54 KB of minima and tables each) hide one another's barriers
    const int g4 = std::max<int>(1, std::min<int64_t>(gmax, (int64_t)(50 * 1024) / ((int64_t)n_hash * 4)));
    for (int g = 1; g <= g4; ++g) {
        if (g * mean < 0.9 * threads && g < g4) continue;  // at least about one round
        const double f = g * mean, hi = f + 1.0 * std::sqrt(f);
        const double eff = f / (threads * std::ceil(hi / threads));
        if (eff > best_eff - 1e-9) {  // ties go to the larger tile (fewer claims and barriers per set)
            best_eff = eff;
            best = g;
        }
    }
    return best;
}

int64_t gap_full_wave_sets(int32_t n_hash, int64_t n_sets, int64_t nnz) {
    if (gap_sets_per_tile(n_hash) < 1 || n_sets < 1) return INT64_MAX;
    return (int64_t)4 * 148 * gap_pick_sets(n_hash, n_sets, nnz, kGapThreads);
}

// The enumeration pays when a feature's N visits cost more than its descent plus its
// ~N c / n hits (9 instructions each; the model's 11.5 allows for a warp's lanes finishing
// apart) and the set's fallback entries.
bool gap_supported(int kind, uint64_t prime, int32_t n_hash, int64_t n_sets, int64_t nnz) {
    if (kind != KIND_ITERATIVE || prime >= (1ull << 31)) return false;
    if (gap_sets_per_tile(n_hash) < 1 || n_sets < 1 || nnz < 1) return false;
    return true;
}

bool gap_preferred(int kind, uint64_t prime, int32_t n_hash, int64_t n_sets, int64_t nnz) {
    const char* env = std::getenv("MHB_GAP");  // read per call: tests and A/B runs switch it
    const int mode = env ? std::atoi(env) : -1;
    if (mode == 0 || !gap_supported(kind, prime, n_hash, n_sets, nnz)) return false;
    if (mode == 1) return true;
    const double mean = (double)nnz / (double)n_sets;
    const double c = std::max(1.0, std::log(0.73 * std::max(mean, 1.0)));
    const double old_cost = 2.7 * n_hash * mean;                         // visits
    const double new_cost = mean * (600.0 + 11.5 * n_hash * c / std::max(mean, 1.0)) +  // descent + hits
                            n_hash * (10.0 + std::exp(-c) * mean * 8.0);                // rows + fallback
    return new_cost * 1.3 < old_cost;
}

int launch_sign_gap(const SignArgs& S, int64_t nnz, int32_t out_dtype, const DeviceInfo& dev, cudaStream_t st) {
    GapArgs A{};
    A.indptr = S.indptr;
    A.ids = S.ids;
    A.n_sets = S.n_sets;
    A.p = S.p;
    A.b = S.b;
    A.a = (uint32_t)(S.ia % S.p);
    A.ap = shoup_companion(A.a, S.p);
    A.n_hash = S.n_hash;
    const char* ce = std::getenv("MHB_GAP_CMUL");
    A.cmul = ce ? (float)std::atof(ce) : 1.0f;
    A.one = 1u;
    A.tab = S.tab;
    A.inv = S.inv;
    A.next = &S.sched->next;
    A.status = S.status;
    A.out = S.out;
    int threads = kGapThreads;
    if (const char* te = std::getenv("MHB_GAP_THREADS")) threads = std::atoi(te);
    if (threads != 64 && threads != 128 && threads != 512) threads = 256;
    A.G = gap_pick_sets(S.n_hash, S.n_sets, nnz, threads);
    if (const char* ge = std::getenv("MHB_GAP_SETS")) A.G = std::max(1, std::min(std::atoi(ge), gap_sets_per_tile(S.n_hash)));
    A.G = std::min(A.G, threads - 1);  // thread g loads set g's offset, thread G the end
    const size_t smem = (size_t)A.G * S.n_hash * 4 + 16;
    const bool reg_inv = threads >= 256 && (S.n_hash & 3) == 0 && S.n_hash <= 8 * 256;
    using Fn = void (*)(GapArgs);
    // lane constants per tile when a tile holds many sets (the reload amortises), for the launch else
    int inv_mode = !reg_inv ? 0 : A.G >= 12 ? 2 : 1;
    if (const char* ie = std::getenv("MHB_GAP_INV")) inv_mode = reg_inv ? std::max(0, std::min(std::atoi(ie), 2)) : 0;
    Fn fn;
    if (out_dtype == MHB_OUT_I64)
        fn = threads == 64    ? (Fn)sign_gap_kernel<long long, 0, 64>
             : threads == 128 ? (Fn)sign_gap_kernel<long long, 0, 128>
             : threads == 512 ? (inv_mode ? (Fn)sign_gap_kernel<long long, 1, 512> : (Fn)sign_gap_kernel<long long, 0, 512>)
             : inv_mode == 2  ? (Fn)sign_gap_kernel<long long, 2, 256>
             : inv_mode == 1  ? (Fn)sign_gap_kernel<long long, 1, 256>
                              : (Fn)sign_gap_kernel<long long, 0, 256>;
    else
        fn = threads == 64    ? (Fn)sign_gap_kernel<uint32_t, 0, 64>
             : threads == 128 ? (Fn)sign_gap_kernel<uint32_t, 0, 128>
             : threads == 512 ? (inv_mode ? (Fn)sign_gap_kernel<uint32_t, 1, 512> : (Fn)sign_gap_kernel<uint32_t, 0, 512>)
             : inv_mode == 2  ? (Fn)sign_gap_kernel<uint32_t, 2, 256>
             : inv_mode == 1  ? (Fn)sign_gap_kernel<uint32_t, 1, 256>
                              : (Fn)sign_gap_kernel<uint32_t, 0, 256>;
    // the attribute and the occupancy query once per (device, kernel, shared-memory size)
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t>, int> occ_of;
    int occ = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        const auto key = std::make_tuple(dev.device, (const void*)fn, smem);
        const auto it = occ_of.find(key);
        if (it != occ_of.end()) {
            occ = it->second;
        } else {
            // the limit is per kernel, not per launch: always the largest tile
            int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)(kGapBestBytes + 16)),
                                "gap kernel shared memory");
            if (rc) return rc;
            rc = cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem), "gap occupancy");
            if (rc) return rc;
            occ_of[key] = occ;
        }
    }
    if (occ < 1) return set_error(MHB_ERR_INVALID, "gap kernel does not fit an SM (n_hash %d)", S.n_hash);
    const int64_t tiles = (S.n_sets + A.G - 1) / A.G;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)occ * dev.sms));
    fn<<<(unsigned)blocks, threads, smem, st>>>(A);
    return cuda_check(cudaGetLastError(), "sign_gap_kernel launch");
}

}  // namespace mhb
