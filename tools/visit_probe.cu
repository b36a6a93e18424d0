// visit_probe.cu -- microbenchmark of the iterative visit sequence (registers only).
//
// Measures visits/clk/SM for walk shapes the signature kernel could use:
//   lanes per thread K, independent feature chains C per thread, and
//   lookahead L (lanes advanced per chain step: L=2 derives h_{i+1}, h_{i+2}
//   both from h_i, halving the dependent chain length).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o visit_probe visit_probe.cu
#include <cstdint>
#include <cstdio>

__device__ uint32_t g_sink;

__device__ __forceinline__ uint32_t red(uint32_t t, uint32_t p) { return __viaddmin_u32(t, 0u - p, t); }
// FMA-pipe-only step: h' = (h + d) mod p from u = h + (d - p): c = umulhi(u, two) is u's
// sign bit (two = 2 passed opaquely so it stays an IMAD.HI), h' = u + c*p.
__device__ __forceinline__ uint32_t step_fma(uint32_t h, uint32_t dm, uint32_t p, uint32_t two) {
    const uint32_t u = h + dm;
    const uint32_t c = __umulhi(u, two);
    return u + c * p;
}

// Lookahead walk where reductions with (j % M == 0) on chain A and (j % M == M/2) on
// chain B go through step_fma; M = 0 disables.
template <int K, int M>
__global__ void __launch_bounds__(256) walk_mixed(int rounds, uint32_t p, uint32_t seed, uint32_t two, long long* cyc) {
    uint32_t best[K];
#pragma unroll
    for (int k = 0; k < K; ++k) best[k] = 0xffffffffu;
    uint32_t h0a = (threadIdx.x * 2654435761u + seed) % p, h0b = (threadIdx.x * 40503u + 7u * seed) % p;
    const uint32_t da = (blockIdx.x * 40503u + 17u + seed) % p, db = (blockIdx.x * 977u + 5u) % p;
    const uint32_t da2 = (2 * da) % p, db2 = (2 * db) % p;
    const uint32_t dam = da - p, dbm = db - p;
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        uint32_t ha = h0a, hb = h0b;
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            const int j = k / 2;
            const bool fa = M > 0 && (j % M == 0), fb = M > 0 && (j % M == M / 2);
            const uint32_t ga = fa ? step_fma(ha, dam, p, two) : red(ha + da, p);
            const uint32_t gb = fb ? step_fma(hb, dbm, p, two) : red(hb + db, p);
            best[k] = __vimin3_u32(best[k], ha, hb);
            best[k + 1] = __vimin3_u32(best[k + 1], ga, gb);
            ha = red(ha + da2, p);
            hb = red(hb + db2, p);
        }
        h0a = red(h0a + (uint32_t)r, p);
        h0b = red(h0b + 3u, p);
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_sink = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Lookahead walk where odd lanes skip the reduction: best = min3(min3(best, t, t-p), u, u-p)
// with t = hA + da, u = hB + db unreduced.  PHI: 1 = every odd lane, 2 = every other odd lane.
__device__ __forceinline__ uint32_t mad1(uint32_t h, uint32_t one, uint32_t d) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(h), "r"(one), "r"(d));
    return r;
}

template <int K, int PHI>
__global__ void __launch_bounds__(256) walk_unred(int rounds, uint32_t p, uint32_t seed, long long* cyc, uint32_t one) {
    uint32_t best[K];
#pragma unroll
    for (int k = 0; k < K; ++k) best[k] = 0xffffffffu;
    uint32_t h0a = (threadIdx.x * 2654435761u + seed) % p, h0b = (threadIdx.x * 40503u + 7u * seed) % p;
    const uint32_t da = (blockIdx.x * 40503u + 17u + seed) % p, db = (blockIdx.x * 977u + 5u) % p;
    const uint32_t da2 = (2 * da) % p, db2 = (2 * db) % p;
    const uint32_t dam = da - p, dbm = db - p;
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        uint32_t ha = h0a, hb = h0b;
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            best[k] = __vimin3_u32(best[k], ha, hb);
            if (PHI > 0 && ((k / 2) % PHI == 0)) {
                best[k + 1] = __vimin3_u32(__vimin3_u32(best[k + 1], mad1(ha, one, da), mad1(ha, one, dam)),
                                           mad1(hb, one, db), mad1(hb, one, dbm));
            } else {
                best[k + 1] = __vimin3_u32(best[k + 1], red(ha + da, p), red(hb + db, p));
            }
            ha = red(ha + da2, p);
            hb = red(hb + db2, p);
        }
        h0a = red(h0a + (uint32_t)r, p);
        h0b = red(h0b + 3u, p);
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_sink = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K, int PHI>
void run_unred(const char* name, int sms, int occ_cap) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk_unred<K, PHI>, 256, 0);
    if (occ > occ_cap) occ = occ_cap;
    int blocks = occ * sms;
    long long* cyc;
    cudaMalloc(&cyc, blocks * sizeof(long long));
    int rounds = 2000;
    walk_unred<K, PHI><<<blocks, 256>>>(rounds / 10, 16777259u, 1u, cyc, 1u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    walk_unred<K, PHI><<<blocks, 256>>>(rounds, 16777259u, 2u, cyc, 1u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    double visits = (double)blocks * 256 * rounds * K * 2;
    printf("%-22s K=%3d PHI=%d occ=%d  %.2f Tvisit/s  %.2f visits/clk/SM\n", name, K, PHI, occ,
           visits / (ms * 1e-3) / 1e12, visits / sms / (double)mx);
    delete[] h;
    cudaFree(cyc);
}

template <int K, int M>
void run_mixed(const char* name, int sms, int occ_cap) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk_mixed<K, M>, 256, 0);
    if (occ > occ_cap) occ = occ_cap;
    int blocks = occ * sms;
    long long* cyc;
    cudaMalloc(&cyc, blocks * sizeof(long long));
    int rounds = 2000;
    walk_mixed<K, M><<<blocks, 256>>>(rounds / 10, 16777259u, 1u, 2u, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    walk_mixed<K, M><<<blocks, 256>>>(rounds, 16777259u, 2u, 2u, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    double visits = (double)blocks * 256 * rounds * K * 2;
    printf("%-22s K=%3d M=%d occ=%d  %.2f Tvisit/s  %.2f visits/clk/SM\n", name, K, M, occ,
           visits / (ms * 1e-3) / 1e12, visits / sms / (double)mx);
    delete[] h;
    cudaFree(cyc);
}

template <int K, int C, int L, bool VECP = false>
__global__ void __launch_bounds__(256) walk(int rounds, uint32_t p_arg, uint32_t seed, long long* cyc, const uint32_t* pv = nullptr) {
    const uint32_t p = VECP ? pv[threadIdx.x] : p_arg;  // VECP: p in a vector register
    uint32_t best[K];
#pragma unroll
    for (int k = 0; k < K; ++k) best[k] = 0xffffffffu;
    uint32_t h0[C], d[C], d2[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        h0[c] = (threadIdx.x * 2654435761u + seed * (c + 1)) % p;
        d[c] = (blockIdx.x * 40503u + 17u * c + seed) % p;
        d2[c] = (2 * d[c]) % p;
    }
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        uint32_t h[C];
#pragma unroll
        for (int c = 0; c < C; ++c) h[c] = h0[c];
        if (L == 1) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (C == 1) best[k] = min(best[k], h[0]);
                if (C >= 2) best[k] = __vimin3_u32(best[k], h[0], h[1]);
                if (C >= 4) best[k] = __vimin3_u32(best[k], h[2], h[3]);
#pragma unroll
                for (int c = 0; c < C; ++c) h[c] = red(h[c] + d[c], p);
            }
        } else if (L == 4) {
            uint32_t d3[C], d4[C];
#pragma unroll
            for (int c = 0; c < C; ++c) { d3[c] = red(d2[c] + d[c], p); d4[c] = red(d2[c] + d2[c], p); }
#pragma unroll
            for (int k = 0; k < K; k += 4) {
                uint32_t g1[C], g2[C], g3[C];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    g1[c] = red(h[c] + d[c], p); g2[c] = red(h[c] + d2[c], p); g3[c] = red(h[c] + d3[c], p);
                }
                if (C >= 2) {
                    best[k] = __vimin3_u32(best[k], h[0], h[1]);
                    best[k + 1] = __vimin3_u32(best[k + 1], g1[0], g1[1]);
                    best[k + 2] = __vimin3_u32(best[k + 2], g2[0], g2[1]);
                    best[k + 3] = __vimin3_u32(best[k + 3], g3[0], g3[1]);
                }
#pragma unroll
                for (int c = 0; c < C; ++c) h[c] = red(h[c] + d4[c], p);
            }
        } else {
#pragma unroll
            for (int k = 0; k < K; k += 2) {
                uint32_t g[C];
#pragma unroll
                for (int c = 0; c < C; ++c) g[c] = red(h[c] + d[c], p);
                if (C == 1) { best[k] = min(best[k], h[0]); best[k + 1] = min(best[k + 1], g[0]); }
                if (C >= 2) {
                    best[k] = __vimin3_u32(best[k], h[0], h[1]);
                    best[k + 1] = __vimin3_u32(best[k + 1], g[0], g[1]);
                }
                if (C >= 4) {
                    best[k] = __vimin3_u32(best[k], h[2], h[3]);
                    best[k + 1] = __vimin3_u32(best[k + 1], g[2], g[3]);
                }
#pragma unroll
                for (int c = 0; c < C; ++c) h[c] = red(h[c] + d2[c], p);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) h0[c] = red(h0[c] + (uint32_t)r, p);
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= best[k];
    if (acc == 0x9e3779b9u) g_sink = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K, int C, int L, bool VECP = false>
void run(const char* name, int sms, int occ_cap = 99) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk<K, C, L, VECP>, 256, 0);
    if (occ > occ_cap) occ = occ_cap;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, walk<K, C, L, VECP>);
    uint32_t* pv;
    cudaMalloc(&pv, 256 * 4);
    uint32_t ph[256];
    for (int i = 0; i < 256; ++i) ph[i] = 16777259u;
    cudaMemcpy(pv, ph, sizeof(ph), cudaMemcpyHostToDevice);
    int blocks = occ * sms;
    long long* cyc;
    cudaMalloc(&cyc, blocks * sizeof(long long));
    int rounds = 2000;
    walk<K, C, L, VECP><<<blocks, 256>>>(rounds / 10, 16777259u, 1u, cyc, pv);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    walk<K, C, L, VECP><<<blocks, 256>>>(rounds, 16777259u, 2u, cyc, pv);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    double visits = (double)blocks * 256 * rounds * K * C;
    double per_sm_clk = visits / sms / (double)mx;
    printf("%-22s K=%3d C=%d L=%d regs=%3d occ=%d warps/SM=%2d  %.2f Tvisit/s  %.2f visits/clk/SM  clk=%.0f MHz\n", name, K,
           C, L, fa.numRegs, occ, occ * 8, visits / (ms * 1e-3) / 1e12, per_sm_clk, mx / (ms * 1e3));
    delete[] h;
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs=%d (ALU-pipe ceiling at 1.5 ALU instr/visit = 42.7 visits/clk/SM)\n", sms);
    run<64, 2, 2>("lookahead occ2", sms, 2);
    run_unred<64, 0>("unred off", sms, 2);
    run_unred<64, 1>("unred all odd", sms, 2);
    run_unred<64, 2>("unred 1/2 odd", sms, 2);
    run_unred<64, 3>("unred 1/3 odd", sms, 2);
    run_mixed<64, 0>("mixed off", sms, 2);
    run_mixed<64, 2>("mixed 1/4", sms, 2);
    run_mixed<64, 3>("mixed 1/6", sms, 2);
    run_mixed<64, 4>("mixed 1/8", sms, 2);
    run_mixed<64, 6>("mixed 1/12", sms, 2);
    run<64, 2, 2, true>("lookahead occ2 vec-p", sms, 2);
    run<64, 2, 4>("lookahead4 occ2", sms, 2);
    run<64, 2, 4>("lookahead4", sms);
    run<32, 2, 2>("lookahead occ3", sms, 3);
    run<32, 2, 4>("lookahead4 occ3", sms, 3);
    run<64, 2, 1>("base", sms);
    run<64, 2, 2>("lookahead", sms);
    run<64, 4, 1>("4 chains", sms);
    run<64, 4, 2>("4 chains lookahead", sms);
    run<32, 2, 1>("base", sms);
    run<32, 2, 2>("lookahead", sms);
    run<32, 4, 1>("4 chains", sms);
    run<32, 4, 2>("4 chains lookahead", sms);
    run<128, 2, 1>("base", sms);
    run<128, 2, 2>("lookahead", sms);
    run<64, 1, 1>("1 chain", sms);
    run<64, 1, 2>("1 chain lookahead", sms);
    return 0;
}
