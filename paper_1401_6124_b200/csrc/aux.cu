// aux.cu -- Jaccard estimates over signature blocks, bucket-uniformity
// histograms, and the visit-rate probe used for the roofline.
//
// Reference:
//   estimate_jaccard   minhash.py:130-137  float(mean(g1.mins == g2.mins))
//   _pair_estimate     bench.py:165-168    same, inline
//   bucket histogram   stats.py:221-224    bincount(family.eval_all(x) % buckets)
#include <cuda_runtime.h>

#include <cstdint>

#include "bandhash.cuh"
#include "common.h"
#include "modarith.cuh"

namespace mhb {

// ---------------------------------------------------------------------------
// Jaccard: listed pairs, one warp per pair
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ uint32_t eq_count16(const uint4& a, const uint4& b) {
    if constexpr (sizeof(T) == 4) {
        return (a.x == b.x) + (a.y == b.y) + (a.z == b.z) + (a.w == b.w);
    } else {  // two int64 entries per 16 bytes
        return ((a.x == b.x) & (a.y == b.y)) + ((a.z == b.z) & (a.w == b.w));
    }
}

// VEC: rows are 16-byte aligned and a whole number of 16-byte words (n_hash*sizeof(T) % 16 == 0):
// each lane compares 16-byte words, four in flight per iteration.
template <typename T, bool VEC>
__global__ void jaccard_pairs_kernel(const T* __restrict__ sig, int32_t n_hash,
                                     const int64_t* __restrict__ pi, const int64_t* __restrict__ pj,
                                     int64_t n_pairs, uint32_t* __restrict__ counts,
                                     double* __restrict__ est) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp0; k < n_pairs; k += nwarps) {
        const T* r1 = sig + pi[k] * (int64_t)n_hash;
        const T* r2 = sig + pj[k] * (int64_t)n_hash;
        uint32_t c = 0;
        if constexpr (VEC) {
            const uint4* v1 = reinterpret_cast<const uint4*>(r1);
            const uint4* v2 = reinterpret_cast<const uint4*>(r2);
            const int nw = (int)((int64_t)n_hash * sizeof(T) / 16);
            int w = lane;
            for (; w + 96 < nw; w += 128) {
                const uint4 a0 = __ldg(v1 + w), a1 = __ldg(v1 + w + 32), a2 = __ldg(v1 + w + 64), a3 = __ldg(v1 + w + 96);
                const uint4 b0 = __ldg(v2 + w), b1 = __ldg(v2 + w + 32), b2 = __ldg(v2 + w + 64), b3 = __ldg(v2 + w + 96);
                c += eq_count16<T>(a0, b0) + eq_count16<T>(a1, b1) + eq_count16<T>(a2, b2) + eq_count16<T>(a3, b3);
            }
            for (; w < nw; w += 32) c += eq_count16<T>(__ldg(v1 + w), __ldg(v2 + w));
        } else {
            for (int32_t i = lane; i < n_hash; i += 32) c += (__ldg(r1 + i) == __ldg(r2 + i));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            counts[k] = c;
            if (est) est[k] = (double)c / (double)n_hash;
        }
    }
}

// ---------------------------------------------------------------------------
// Jaccard: block x block, 32x32 output tile per CTA, hash dimension staged in smem
// ---------------------------------------------------------------------------
template <typename T>
__global__ void jaccard_block_kernel(const T* __restrict__ A, int64_t n_rows, const T* __restrict__ B,
                                     int64_t n_cols, int32_t n_hash, uint32_t* __restrict__ counts) {
    constexpr int TILE = 32, HC = 32;
    __shared__ T sa[TILE][HC + 1];
    __shared__ T sb[TILE][HC + 1];
    const int tx = threadIdx.x & 31;  // column within tile
    const int ty = threadIdx.x >> 5;  // 8 warps -> 4 rows each
    const int64_t r0 = (int64_t)blockIdx.y * TILE, c0 = (int64_t)blockIdx.x * TILE;
    uint32_t acc[4] = {0, 0, 0, 0};
    for (int32_t h0 = 0; h0 < n_hash; h0 += HC) {
        for (int t = threadIdx.x; t < TILE * HC; t += blockDim.x) {
            const int rr = t / HC, hh = t % HC;
            const int64_t gr = r0 + rr, gc = c0 + rr;
            const int32_t gh = h0 + hh;
            sa[rr][hh] = (gr < n_rows && gh < n_hash) ? A[gr * n_hash + gh] : (T)-1;
            sb[rr][hh] = (gc < n_cols && gh < n_hash) ? B[gc * n_hash + gh] : (T)-2;
        }
        __syncthreads();
        const int hn = (n_hash - h0) < HC ? (n_hash - h0) : HC;
        for (int hh = 0; hh < hn; ++hh) {
            const T bv = sb[tx][hh];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += (sa[ty * 4 + q][hh] == bv);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t r = r0 + ty * 4 + q, c = c0 + tx;
        if (r < n_rows && c < n_cols) counts[r * n_cols + c] = acc[q];
    }
}

// ---------------------------------------------------------------------------
// Bucket histogram (stats.py:221-224 generalised to a batch of x): counts[b] =
// #{(x, i) : h_i(x) mod m = b}.
//
// One count per (x, i) evaluation, so the counting instruction is the kernel.  Round 1
// counted into one CTA-wide u32 table with shared atomics: uniform bins over 4096
// entries put ~3.5 lanes of a warp on one bank (4.7 counts/clk/SM).  hist_kernel8
// gives each lane slot s = lane % (2 COLS) its own 16-bit counter per bin: bin b,
// slot s lives in word b * COLS + (s % COLS), half s / COLS.  So
//   * a lane's increment is a per-lane constant (1 or 1 << 16) and its address one
//     LOP3 + IMAD from h: walk (2) + address (2) + RED = 5 instructions per evaluation;
//   * a warp's 32 increments spread over the banks by column: the 32 / COLS lanes of
//     one column share 32 / COLS banks (COLS = 8: ~2 lanes per bank at worst, against
//     ~3.5 for one table; tools/atoms_probe.cu measures the RED rates);
//   * 4096 bins x 2 COLS slots x 2 B + a 16 KB u32 table fit one SM (COLS = 8: 144 KB,
//     1024 threads; COLS = 4: 80 KB, two CTAs of 512).
// A counter is shared by the lanes of its slot in every warp of the CTA (64 threads),
// so the CTA sweeps the counters into the u32 table before any can pass 65535: every
// thread runs the same rounds of at most 2 x `run` evaluations (two x per round, two
// independent dependency chains), and the CTA sweeps every floor(65535 / 64 / 2 run)
// rounds.  cfg3 (4.19M ids x 512): 1.56 -> 0.58 ms; cfg4 (60.9M x 2048): 91.5 -> 34.3 ms.
// ---------------------------------------------------------------------------
constexpr int kRun = 256;
// COLS word columns per bin (2 x 16-bit slots each): 8 for the iterative walk (128 KB,
// one CTA of 1024 threads per SM: 4 lanes per column, fewer bank collisions), 4 for
// the random family (64 KB, two CTAs of 512: its 48 lane constants need the registers).
constexpr int kRepMaxBins = 4096;  // 4096 x COLS words + a 4096-word u32 table
template <int COLS>
struct HistShape {
    static constexpr int threads = COLS == 4 ? 512 : 1024;
    static constexpr int sharers = (32 / (2 * COLS)) * (threads / 32);  // threads per 16-bit counter
    static constexpr int max_run = 65535 / sharers;                     // evaluations per thread per sweep
};

struct HistArgs {
    const uint32_t* xs;
    int64_t n_x;
    uint32_t p, b;
    uint64_t a;
    int32_t n_hash;
    uint32_t m, mp;  // buckets, floor(2^32 / m) (m >= 2)
    const uint32_t* ra;
    const uint32_t* rb;
    unsigned long long* counts;
    int kind;
    int use_smem;
    int nblk, run;   // hist_kernel8: lane blocks per x (power of two) and lanes per block
};

__device__ __forceinline__ uint32_t mod_bucket(uint32_t h, uint32_t m, uint32_t mp) {
    if (m == 1) return 0;
    uint32_t r = h - __umulhi(h, mp) * m;  // in [0, 2m)
    return __viaddmin_u32(r, 0u - m, r);
}

__device__ __forceinline__ void reds_add(uint32_t saddr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

// One evaluation's count: this lane's counter for bin h mod m (`col` = shared address of
// the lane's word column, `inc` = its half).
template <bool POW2, int COLS>
__device__ __forceinline__ void count_bin(uint32_t col, uint32_t inc, uint32_t h, uint32_t m, uint32_t mp) {
    const uint32_t bin = POW2 ? (h & (m - 1)) : mod_bucket(h, m, mp);
    reds_add(bin * (4u * COLS) + col, inc);
}

// Move the 16-bit counters into the u32 table and clear them.  Thread t owns bins
// b = t, t + blockDim, ... (exclusive: plain adds): one 16-byte load holds all 8 slots.
template <int COLS>
__device__ __forceinline__ void sweep8(uint4* cnt, uint32_t* acc, uint32_t m) {
    for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < COLS / 4; ++q) {
            const uint4 v = cnt[b * (COLS / 4) + q];
            cnt[b * (COLS / 4) + q] = make_uint4(0u, 0u, 0u, 0u);
            sum += (v.x & 0xFFFFu) + (v.x >> 16) + (v.y & 0xFFFFu) + (v.y >> 16) + (v.z & 0xFFFFu) + (v.z >> 16) +
                   (v.w & 0xFFFFu) + (v.w >> 16);
        }
        acc[b] += sum;
    }
}

template <bool ITER, bool POW2, int RL, int COLS>
__global__ void __launch_bounds__(HistShape<COLS>::threads) hist_kernel8(HistArgs H) {
    extern __shared__ uint4 smem4[];
    const uint32_t m = H.m;
    uint4* cnt = smem4;                                                      // [m] x 2*COLS slots (16-bit)
    uint32_t* acc = reinterpret_cast<uint32_t*>(smem4 + m * (COLS / 4));  // [m] u32
    for (uint32_t i = threadIdx.x; i < m * (COLS / 4); i += blockDim.x) cnt[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) acc[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t col = (uint32_t)__cvta_generic_to_shared(cnt) + 4u * (uint32_t)(lane & (COLS - 1));
    const uint32_t inc = (lane & COLS) ? 0x10000u : 1u;
    const uint32_t p = H.p, mp = H.mp;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;  // a multiple of nblk
    // this thread's lane block is fixed: units u = gtid + k * nthreads, blk = u % nblk
    const int blk = (int)(gtid & (H.nblk - 1));
    const int32_t i0 = blk * H.run;
    const int32_t i1 = min(i0 + H.run, H.n_hash);
    const int n = i1 - i0;
    const int64_t xstride = nthreads / H.nblk;
    // rounds of two x each; every thread of the CTA runs its first thread's count (the most)
    const int64_t x_first = ((int64_t)blockIdx.x * blockDim.x) / H.nblk;
    const int64_t rounds = x_first < H.n_x ? (H.n_x - x_first + 2 * xstride - 1) / (2 * xstride) : 0;
    const int per_sweep = HistShape<COLS>::max_run / (2 * (H.run > 0 ? H.run : 1));
    int64_t xi = gtid / H.nblk;

    uint32_t A = 0, Ap = 0, B = 0;
    uint32_t cA[RL], cAp[RL], cB[RL];
    if (ITER) {
        // h_{i0}(x) = (a + i0) x + i0 b mod p (families.py:170-176), then the additive walk
        A = (uint32_t)((H.a + (uint64_t)i0) % p);
        Ap = shoup_companion(A, p);
        B = (uint32_t)((uint64_t)i0 * H.b % p);
    } else {
#pragma unroll
        for (int k = 0; k < RL; ++k) {
            const int32_t i = min(i0 + k, H.n_hash - 1);
            cA[k] = H.ra[i];
            cAp[k] = shoup_companion(cA[k], p);
            cB[k] = H.rb[i];
        }
    }
    const bool narrow = 3ull * p < (1ull << 32);
    // next round's x prefetched (an L2 round trip per round otherwise)
    uint32_t xa_n = xi < H.n_x ? __ldg(H.xs + xi) : 0u;
    uint32_t xb_n = xi + xstride < H.n_x ? __ldg(H.xs + xi + xstride) : 0u;
    for (int64_t r0 = 0; r0 < rounds; r0 += per_sweep) {
        const int64_t r1 = min(rounds, r0 + per_sweep);
        for (int64_t r = r0; r < r1; ++r, xi += 2 * xstride) {
            const uint32_t xa = xa_n, xb = xb_n;
            const bool va = xi < H.n_x && n > 0, vb = xi + xstride < H.n_x && n > 0;
            const int64_t xn = xi + 2 * xstride;
            xa_n = xn < H.n_x ? __ldg(H.xs + xn) : 0u;
            xb_n = xn + xstride < H.n_x ? __ldg(H.xs + xn + xstride) : 0u;
            if (ITER) {
                if (va && vb) {
                    uint32_t ha = mul_add_mod(A, Ap, B, xa, p), hb = mul_add_mod(A, Ap, B, xb, p);
                    const uint32_t da = reduce_once(xa + H.b, p), db = reduce_once(xb + H.b, p);
#pragma unroll 2
                    for (int k = 0; k < n; ++k) {
                        count_bin<POW2, COLS>(col, inc, ha, m, mp);
                        count_bin<POW2, COLS>(col, inc, hb, m, mp);
                        ha = reduce_once(ha + da, p);
                        hb = reduce_once(hb + db, p);
                    }
                } else if (va) {
                    uint32_t ha = mul_add_mod(A, Ap, B, xa, p);
                    const uint32_t da = reduce_once(xa + H.b, p);
                    for (int k = 0; k < n; ++k) {
                        count_bin<POW2, COLS>(col, inc, ha, m, mp);
                        ha = reduce_once(ha + da, p);
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t x = e ? xb : xa;
                    if (!(e ? vb : va)) continue;
                    if (n == RL && narrow) {
                        // random family: RL lanes' constants in registers, one Shoup multiply-add each
#pragma unroll
                        for (int k = 0; k < RL; ++k)
                            count_bin<POW2, COLS>(col, inc, mul_add_mod_narrow(cA[k], cAp[k], cB[k], x, p), m, mp);
                    } else {
#pragma unroll
                        for (int k = 0; k < RL; ++k)
                            if (k < n) count_bin<POW2, COLS>(col, inc, mul_add_mod(cA[k], cAp[k], cB[k], x, p), m, mp);
                    }
                }
            }
        }
        __syncthreads();
        sweep8<COLS>(cnt, acc, m);
        __syncthreads();
    }
    for (uint32_t bin = threadIdx.x; bin < m; bin += blockDim.x)
        if (acc[bin]) atomicAdd(H.counts + bin, (unsigned long long)acc[bin]);
}

// Fallback for m > 4096 (or p >= 2^31 is handled below): one u32 table per CTA in
// shared memory when it fits, else global atomics.
__global__ void hist_kernel(HistArgs H) {
    extern __shared__ uint32_t bins[];
    if (H.use_smem) {
        for (uint32_t i = threadIdx.x; i < H.m; i += blockDim.x) bins[i] = 0;
        __syncthreads();
    }
    const int64_t runs_per_x = (H.n_hash + kRun - 1) / kRun;
    const int64_t units = H.n_x * runs_per_x;
    const uint32_t p = H.p;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xi = u / runs_per_x;
        const int32_t i0 = (int32_t)(u - xi * runs_per_x) * kRun;
        const int32_t i1 = min(i0 + kRun, H.n_hash);
        const uint32_t x = H.xs[xi];
        if (H.kind == 0) {
            const uint32_t A = (uint32_t)((H.a + (uint64_t)i0) % p);
            const uint32_t B = (uint32_t)((uint64_t)i0 * H.b % p);
            uint32_t h = mul_add_mod(A, shoup_companion(A, p), B, x, p);
            const uint32_t dh = reduce_once(x + H.b, p);
            for (int32_t i = i0; i < i1; ++i) {
                const uint32_t bin = mod_bucket(h, H.m, H.mp);
                if (H.use_smem) atomicAdd(&bins[bin], 1u);
                else atomicAdd(&H.counts[bin], 1ull);
                h = reduce_once(h + dh, p);
            }
        } else {
            for (int32_t i = i0; i < i1; ++i) {
                const uint32_t a = H.ra[i];
                const uint32_t h = mul_add_mod(a, shoup_companion(a, p), H.rb[i], x, p);
                const uint32_t bin = mod_bucket(h, H.m, H.mp);
                if (H.use_smem) atomicAdd(&bins[bin], 1u);
                else atomicAdd(&H.counts[bin], 1ull);
            }
        }
    }
    if (H.use_smem) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < H.m; i += blockDim.x)
            if (bins[i]) atomicAdd(&H.counts[i], (unsigned long long)bins[i]);
    }
}

// Primes 2^31 <= p < 2^63 (the reference counts for any prime, families.py:105-112):
// 64-bit residues with 128-bit products, global atomics.  Correctness path.
__device__ __forceinline__ uint64_t hist_mulmod64(uint64_t a, uint64_t b, uint64_t p) {
    return (uint64_t)(((unsigned __int128)a * b) % p);
}

template <typename IdT>
__global__ void hist_wide_kernel(const IdT* __restrict__ xs, int64_t n_x, int kind, uint64_t a, uint64_t b,
                                 const uint64_t* __restrict__ ra, const uint64_t* __restrict__ rb, uint64_t p,
                                 int32_t n_hash, uint64_t m, unsigned long long* __restrict__ counts) {
    const int64_t runs_per_x = (n_hash + kRun - 1) / kRun;
    const int64_t units = n_x * runs_per_x;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xi = u / runs_per_x;
        const int32_t i0 = (int32_t)(u - xi * runs_per_x) * kRun;
        const int32_t i1 = min(i0 + kRun, n_hash);
        const uint64_t x = (uint64_t)xs[xi];
        if (kind == 0) {
            uint64_t h = (hist_mulmod64((a + (uint64_t)i0) % p, x, p) + hist_mulmod64((uint64_t)i0, b, p)) % p;
            uint64_t dh = x + b;  // x, b < p < 2^63
            if (dh >= p) dh -= p;
            for (int32_t i = i0; i < i1; ++i) {
                atomicAdd(&counts[h % m], 1ull);
                h += dh;
                if (h >= p) h -= p;
            }
        } else {
            for (int32_t i = i0; i < i1; ++i) {
                uint64_t h = hist_mulmod64(ra[i], x, p) + rb[i];
                if (h >= p) h -= p;
                atomicAdd(&counts[h % m], 1ull);
            }
        }
    }
}

template <bool ITER, bool POW2>
static int launch_rep(HistArgs H, const DeviceInfo& dev, cudaStream_t st) {
    constexpr int RL = ITER ? 1 : 16;
    constexpr int COLS = ITER ? 8 : 4;
    using S = HistShape<COLS>;
    auto fn = hist_kernel8<ITER, POW2, RL, COLS>;
    const size_t smem = (size_t)H.m * (COLS * sizeof(uint32_t) + sizeof(uint32_t));
    static int attr_done[64] = {0};
    if (dev.device >= 0 && dev.device < 64 && !attr_done[dev.device]) {
        const int most = kRepMaxBins * (int)(COLS * sizeof(uint32_t) + sizeof(uint32_t));
        int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, most),
                            "hist smem attr");
        if (rc) return rc;
        attr_done[dev.device] = 1;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, S::threads, smem) != cudaSuccess || occ < 1)
        occ = 1;
    // lane blocks per x: a power of two (so the grid's thread count is a multiple of it)
    // with about 64 lanes each for the iterative walk, RL for the random family
    const int want = ITER ? (H.n_hash + 63) / 64 : (H.n_hash + RL - 1) / RL;
    int nblk = 1;
    while (nblk < want && nblk < 512) nblk *= 2;
    H.nblk = nblk;
    H.run = (H.n_hash + nblk - 1) / nblk;
    if (2 * H.run > S::max_run || (!ITER && H.run > RL))
        return set_error(MHB_ERR_UNSUPPORTED, "histogram over %d members needs the fallback kernel", H.n_hash);
    int64_t blocks = (int64_t)occ * dev.sms;
    const int64_t need = (H.n_x * nblk + 2 * S::threads - 1) / (2 * S::threads);  // two x per thread
    if (blocks > need) blocks = need < 1 ? 1 : need;
    fn<<<(unsigned)blocks, S::threads, smem, st>>>(H);
    return cuda_check(cudaGetLastError(), "hist_kernel8 launch");
}

static int launch_hist(HistArgs H, cudaStream_t st) {
    clear_error();
    if (H.m < 1) return set_error(MHB_ERR_INVALID, "need at least one bucket, got %u", H.m);
    if (H.n_hash < 1) return set_error(MHB_ERR_INVALID, "need at least one hash function");
    if (H.p < 3 || !is_prime_u64(H.p)) return set_error(MHB_ERR_INVALID, "modulus %u is not prime", H.p);
    if (H.n_x <= 0) return MHB_OK;
    H.mp = H.m >= 2 ? (uint32_t)((1ull << 32) / H.m) : 0;
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    const bool pow2 = H.m >= 2 && (H.m & (H.m - 1)) == 0;
    const bool rep_ok = H.m <= (uint32_t)kRepMaxBins && (H.kind == 0 ? H.n_hash <= 512 * (HistShape<8>::max_run / 2) : H.n_hash <= 512 * 16);
    if (rep_ok) {
        if (H.kind == 0) return pow2 ? launch_rep<true, true>(H, dev, st) : launch_rep<true, false>(H, dev, st);
        return pow2 ? launch_rep<false, true>(H, dev, st) : launch_rep<false, false>(H, dev, st);
    }
    size_t smem = (size_t)H.m * sizeof(uint32_t);
    H.use_smem = smem <= 96 * 1024;
    if (!H.use_smem) smem = 0;
    if (smem > 48 * 1024) {
        rc = cuda_check(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem), "hist smem attr");
        if (rc) return rc;
    }
    const int64_t units = H.n_x * ((H.n_hash + kRun - 1) / kRun);
    int64_t blocks = (units + 255) / 256;
    if (blocks > (int64_t)dev.sms * 2) blocks = (int64_t)dev.sms * 2;
    if (blocks < 1) blocks = 1;
    hist_kernel<<<(unsigned)blocks, 256, smem, st>>>(H);
    return cuda_check(cudaGetLastError(), "hist_kernel launch");
}

template <typename IdT>
static int launch_hist_wide(const IdT* xs, int64_t n_x, int kind, uint64_t a, uint64_t b, const uint64_t* ra,
                            const uint64_t* rb, uint64_t p, int32_t n_hash, uint64_t m,
                            unsigned long long* counts, cudaStream_t st) {
    if (n_x <= 0) return MHB_OK;
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    const int64_t units = n_x * ((n_hash + kRun - 1) / kRun);
    int64_t blocks = (units + 255) / 256;
    if (blocks > (int64_t)dev.sms * 8) blocks = (int64_t)dev.sms * 8;
    if (blocks < 1) blocks = 1;
    hist_wide_kernel<IdT><<<(unsigned)blocks, 256, 0, st>>>(xs, n_x, kind, a, b, ra, rb, p, n_hash, m, counts);
    return cuda_check(cudaGetLastError(), "hist_wide_kernel launch");
}

// ---------------------------------------------------------------------------
// LSH band keys (bandhash.cuh): one thread per (set, band).
template <typename T>
__global__ void band_keys_kernel(const T* __restrict__ sig, int64_t n_sets, int32_t n_hash, int32_t rows,
                                 int32_t n_bands, unsigned long long* __restrict__ keys) {
    const int64_t total = n_sets * (int64_t)n_bands;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / n_bands;
        const int band = (int)(t - s * n_bands);
        const T* row = sig + s * (int64_t)n_hash + (int64_t)band * rows;
        BandHash h((uint32_t)band);
        for (int j = 0; j < rows; ++j) h.add((uint32_t)__ldg(row + j));
        keys[t] = h.key();
    }
}

// uint32 signatures with rows % 4 == 0 and n_hash % 4 == 0: each band is read with
// rows/4 16-byte loads (the scalar loop issues one 4-byte load per row, and every warp
// load then touches 32 separate 64-byte band spans: L1-wavefront bound, not HBM).
__global__ void band_keys_vec4_kernel(const uint32_t* __restrict__ sig, int64_t n_sets, int32_t n_hash,
                                      int32_t rows, int32_t n_bands, unsigned long long* __restrict__ keys) {
    const int64_t total = n_sets * (int64_t)n_bands;
    const int q = rows >> 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / n_bands;
        const int band = (int)(t - s * n_bands);
        const uint4* row = reinterpret_cast<const uint4*>(sig + s * (int64_t)n_hash + (int64_t)band * rows);
        BandHash h((uint32_t)band);
        for (int j = 0; j < q; ++j) {
            const uint4 v = __ldg(row + j);
            h.add(v.x);
            h.add(v.y);
            h.add(v.z);
            h.add(v.w);
        }
        keys[t] = h.key();
    }
}

// ---------------------------------------------------------------------------
// Visit-rate probe: the iterative inner loop from registers only.
// ---------------------------------------------------------------------------
__device__ uint32_t g_probe_sink;

// The same two-feature lookahead walk as sign.cu walk2_iter (h_{k+1} and h_{k+2} both
// from h_k), so the probe is the register-only ceiling of the kernel's own visit
// sequence (tools/visit_probe.cu "lookahead": 41.9 visits/clk/SM).
template <int K>
__global__ void __launch_bounds__(256) probe_iter_kernel(int64_t rounds, uint32_t p, uint32_t seed) {
    uint32_t best[K];
#pragma unroll
    for (int k = 0; k < K; ++k) best[k] = 0xffffffffu;
    uint32_t h0a = (threadIdx.x * 2654435761u + seed) % p, h0b = (threadIdx.x * 40503u + 7u * seed) % p;
    const uint32_t da = (blockIdx.x * 40503u + 17u + seed) % p, db = (blockIdx.x * 977u + 5u) % p;
    const uint32_t da2 = (2 * da) % p, db2 = (2 * db) % p;
    for (int64_t r = 0; r < rounds; ++r) {
        uint32_t ha = h0a, hb = h0b;
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            const uint32_t ga = reduce_once(ha + da, p), gb = reduce_once(hb + db, p);
            best[k] = __vimin3_u32(best[k], ha, hb);
            best[k + 1] = __vimin3_u32(best[k + 1], ga, gb);
            ha = reduce_once(ha + da2, p);
            hb = reduce_once(hb + db2, p);
        }
        h0a = reduce_once(h0a + (uint32_t)r, p);  // new start hashes per round (not foldable)
        h0b = reduce_once(h0b + 3u, p);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_probe_sink = acc;
}

template <int K>
__global__ void __launch_bounds__(256) probe_random_kernel(int64_t rounds, uint32_t p, uint32_t seed) {
    uint32_t best[K], cA[K], cAp[K], cB[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        best[k] = 0xffffffffu;
        cA[k] = (seed + 977u * k + threadIdx.x) % (p - 1) + 1;
        cAp[k] = (uint32_t)(((uint64_t)cA[k] << 32) / p);
        cB[k] = (seed * 31u + k) % p;
    }
    uint32_t xa = (threadIdx.x * 2654435761u + seed) % p, xb = (xa * 7u + 13u) % p;
    for (int64_t r = 0; r < rounds; ++r) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            best[k] = __vimin3_u32(best[k], mul_add_mod_narrow(cA[k], cAp[k], cB[k], xa, p),
                                   mul_add_mod_narrow(cA[k], cAp[k], cB[k], xb, p));
        xa = reduce_once(xa + 1u, p);
        xb = reduce_once(xb + 3u, p);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_probe_sink = acc;
}

// The random family's float-quotient visit (sign.cu walk2_random_fpq, p <= 2^23), K lanes.
template <int K>
__global__ void __launch_bounds__(256) probe_random_fpq_kernel(int64_t rounds, uint32_t p, uint32_t seed) {
    uint32_t best[K], cA[K], cW[K], cC[K];
    const uint32_t negp = 0u - p;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        best[k] = 0xffffffffu;
        cA[k] = (seed + 977u * k + threadIdx.x) % (p - 1) + 1;
        cW[k] = __float_as_uint(__double2float_rd((double)cA[k] / (double)p));
        cC[k] = (seed * 31u + k) % p + 0x4B000000u * p;
    }
    uint32_t xa = (threadIdx.x * 2654435761u + seed) % p, xb = (xa * 7u + 13u) % p;
    for (int64_t r = 0; r < rounds; ++r) {
        const float fa = __uint2float_rn(xa), fb = __uint2float_rn(xb);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float wf = __uint_as_float(cW[k]);
            const uint32_t qa = __float_as_uint(__fmaf_rz(fa, wf, 8388608.0f));
            const uint32_t qb = __float_as_uint(__fmaf_rz(fb, wf, 8388608.0f));
            const uint32_t ra = reduce_once(reduce_once(cA[k] * xa + cC[k] + qa * negp, p), p);
            const uint32_t rb = reduce_once(reduce_once(cA[k] * xb + cC[k] + qb * negp, p), p);
            best[k] = __vimin3_u32(best[k], ra, rb);
        }
        xa = reduce_once(xa + 1u, p);
        xb = reduce_once(xb + 3u, p);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_probe_sink = acc;
}

}  // namespace mhb

using namespace mhb;

extern "C" int mhb_jaccard_pairs(const void* sig, int32_t sig_dtype, int32_t n_hash, const int64_t* pi,
                                 const int64_t* pj, int64_t n_pairs, uint32_t* counts, double* est,
                                 void* stream) {
    clear_error();
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "signature lengths must be positive");
    if (n_pairs <= 0) return MHB_OK;
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t blocks = (n_pairs * 32 + 255) / 256;
    if (blocks > (int64_t)dev.sms * 16) blocks = (int64_t)dev.sms * 16;
    const size_t esz = sig_dtype == MHB_OUT_I64 ? 8 : 4;
    const bool vec = ((uintptr_t)sig % 16 == 0) && (((size_t)n_hash * esz) % 16 == 0);
    if (sig_dtype == MHB_OUT_I64) {
        const long long* s = static_cast<const long long*>(sig);
        if (vec) jaccard_pairs_kernel<long long, true><<<(unsigned)blocks, 256, 0, st>>>(s, n_hash, pi, pj, n_pairs, counts, est);
        else jaccard_pairs_kernel<long long, false><<<(unsigned)blocks, 256, 0, st>>>(s, n_hash, pi, pj, n_pairs, counts, est);
    } else if (sig_dtype == MHB_OUT_U32) {
        const uint32_t* s = static_cast<const uint32_t*>(sig);
        if (vec) jaccard_pairs_kernel<uint32_t, true><<<(unsigned)blocks, 256, 0, st>>>(s, n_hash, pi, pj, n_pairs, counts, est);
        else jaccard_pairs_kernel<uint32_t, false><<<(unsigned)blocks, 256, 0, st>>>(s, n_hash, pi, pj, n_pairs, counts, est);
    } else {
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    }
    return cuda_check(cudaGetLastError(), "jaccard_pairs launch");
}

extern "C" int mhb_jaccard_block(const void* sig_a, int64_t n_rows, const void* sig_b, int64_t n_cols,
                                 int32_t sig_dtype, int32_t n_hash, uint32_t* counts, void* stream) {
    clear_error();
    if (n_hash < 1) return set_error(MHB_ERR_INVALID, "signature lengths must be positive");
    if (n_rows <= 0 || n_cols <= 0) return MHB_OK;
    if ((n_rows + 31) / 32 > 65535) return set_error(MHB_ERR_INVALID, "n_rows too large for one call");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dim3 grid((unsigned)((n_cols + 31) / 32), (unsigned)((n_rows + 31) / 32));
    if (sig_dtype == MHB_OUT_I64)
        jaccard_block_kernel<long long><<<grid, 256, 0, st>>>(static_cast<const long long*>(sig_a), n_rows,
                                                              static_cast<const long long*>(sig_b), n_cols,
                                                              n_hash, counts);
    else if (sig_dtype == MHB_OUT_U32)
        jaccard_block_kernel<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(sig_a), n_rows,
                                                             static_cast<const uint32_t*>(sig_b), n_cols,
                                                             n_hash, counts);
    else
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    return cuda_check(cudaGetLastError(), "jaccard_block launch");
}

extern "C" int mhb_band_keys(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                             int32_t rows_per_band, unsigned long long* keys, void* stream) {
    clear_error();
    if (n_hash < 1 || rows_per_band < 1 || n_hash % rows_per_band != 0)
        return set_error(MHB_ERR_INVALID, "rows_per_band must divide n_hash (got %d, %d)", rows_per_band, n_hash);
    if (n_sets <= 0) return MHB_OK;
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    const int32_t n_bands = n_hash / rows_per_band;
    int64_t blocks = (n_sets * n_bands + 255) / 256;
    if (blocks > (int64_t)dev.sms * 16) blocks = (int64_t)dev.sms * 16;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sig_dtype == MHB_OUT_I64)
        band_keys_kernel<long long><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const long long*>(sig), n_sets, n_hash,
                                                                      rows_per_band, n_bands, keys);
    else if (sig_dtype == MHB_OUT_U32 && rows_per_band % 4 == 0 && n_hash % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(sig) & 15) == 0)
        band_keys_vec4_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint32_t*>(sig), n_sets, n_hash,
                                                                rows_per_band, n_bands, keys);
    else if (sig_dtype == MHB_OUT_U32)
        band_keys_kernel<uint32_t><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint32_t*>(sig), n_sets, n_hash,
                                                                     rows_per_band, n_bands, keys);
    else
        return set_error(MHB_ERR_INVALID, "unknown sig_dtype %d", sig_dtype);
    return cuda_check(cudaGetLastError(), "band_keys launch");
}

extern "C" int mhb_bucket_hist_iterative(const uint32_t* xs, int64_t n_x, uint64_t a, uint64_t b,
                                         uint64_t prime, int32_t n_hash, uint32_t buckets,
                                         unsigned long long* counts, void* stream) {
    clear_error();
    if (a < 1 || a >= prime || b >= prime || a + (uint64_t)n_hash >= prime)
        return set_error(MHB_ERR_INVALID, "iterative parameters out of range");
    if (prime >= (1ull << 31)) {
        if (buckets < 1 || n_hash < 1) return set_error(MHB_ERR_INVALID, "need buckets >= 1 and n_hash >= 1");
        if (prime >= (1ull << 63) || !is_prime_u64(prime))
            return set_error(MHB_ERR_INVALID, "modulus %llu is not a prime below 2^63", (unsigned long long)prime);
        return launch_hist_wide<uint32_t>(xs, n_x, 0, a, b, nullptr, nullptr, prime, n_hash, buckets, counts,
                                          static_cast<cudaStream_t>(stream));
    }
    HistArgs H{};
    H.xs = xs; H.n_x = n_x; H.p = (uint32_t)prime; H.b = (uint32_t)b; H.a = a;
    H.n_hash = n_hash; H.m = buckets; H.counts = counts; H.kind = 0;
    return launch_hist(H, static_cast<cudaStream_t>(stream));
}

extern "C" int mhb_bucket_hist_random(const uint32_t* xs, int64_t n_x, const uint32_t* a, const uint32_t* b,
                                      uint64_t prime, int32_t n_hash, uint32_t buckets,
                                      unsigned long long* counts, void* stream) {
    clear_error();
    if (prime >= (1ull << 31))
        return set_error(MHB_ERR_UNSUPPORTED, "prime >= 2^31: random-family parameters need 64 bits, use "
                                              "mhb_bucket_hist_u64");
    HistArgs H{};
    H.xs = xs; H.n_x = n_x; H.p = (uint32_t)prime; H.n_hash = n_hash; H.m = buckets;
    H.ra = a; H.rb = b; H.counts = counts; H.kind = 1;
    return launch_hist(H, static_cast<cudaStream_t>(stream));
}

extern "C" int mhb_bucket_hist_u64(int32_t kind, const uint64_t* xs, int64_t n_x, uint64_t a, uint64_t b,
                                   const uint64_t* ra, const uint64_t* rb, uint64_t prime, int32_t n_hash,
                                   uint64_t buckets, unsigned long long* counts, void* stream) {
    clear_error();
    if (kind != 0 && kind != 1) return set_error(MHB_ERR_INVALID, "unknown kind %d", kind);
    if (buckets < 1 || n_hash < 1) return set_error(MHB_ERR_INVALID, "need buckets >= 1 and n_hash >= 1");
    if (prime < 3 || prime >= (1ull << 63) || !is_prime_u64(prime))
        return set_error(MHB_ERR_INVALID, "modulus %llu is not a prime below 2^63", (unsigned long long)prime);
    if (kind == 0 && (a < 1 || a >= prime || b >= prime || a + (uint64_t)n_hash >= prime))
        return set_error(MHB_ERR_INVALID, "iterative parameters out of range");
    if (kind == 1 && (!ra || !rb)) return set_error(MHB_ERR_INVALID, "random family needs device arrays a and b");
    return launch_hist_wide<uint64_t>(xs, n_x, kind, a, b, ra, rb, prime, n_hash, buckets, counts,
                                      static_cast<cudaStream_t>(stream));
}

extern "C" int mhb_probe_visit_rate(int64_t visits_per_thread, int32_t kind, double* visits_out,
                                    float* ms_out, void* stream) {
    clear_error();
    DeviceInfo dev;
    int rc = current_device_info(&dev);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // kind 0: iterative walk (K=64); 1: random family, Shoup lanes (K=64); 2: random family,
    // float-quotient lanes as the kernel runs them for p <= 2^23 (K=16, p = 4,194,319)
    const int K = kind == 2 ? 16 : 64;
    const int64_t rounds = visits_per_thread / (2 * K) > 0 ? visits_per_thread / (2 * K) : 1;
    int occ = 0;
    const void* fn = kind == 0 ? (const void*)probe_iter_kernel<64>
                               : kind == 1 ? (const void*)probe_random_kernel<64> : (const void*)probe_random_fpq_kernel<16>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0);
    if (occ < 1) occ = 1;
    const int blocks = occ * dev.sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&](int64_t r, uint32_t seed) {
        if (kind == 0) probe_iter_kernel<64><<<blocks, 256, 0, st>>>(r, 16777259u, seed);
        else if (kind == 1) probe_random_kernel<64><<<blocks, 256, 0, st>>>(r, 16777259u, seed);
        else probe_random_fpq_kernel<16><<<blocks, 256, 0, st>>>(r, 4194319u, seed);
    };
    launch(rounds / 10 + 1, 1u);  // warm-up
    cudaEventRecord(e0, st);
    launch(rounds, 2u);
    cudaEventRecord(e1, st);
    rc = cuda_check(cudaEventSynchronize(e1), "probe sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    if (visits_out) *visits_out = (double)blocks * 256.0 * (double)rounds * 2.0 * K;
    if (ms_out) *ms_out = ms;
    return MHB_OK;
}
