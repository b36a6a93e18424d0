// walk_mix_probe.cu -- register-only timing of iterative-walk instruction mixes.
//
// The committed walk (walk2_iter) costs per visit: 1 IMAD.IADD (FMA pipe, immediate
// form) + 1 VIADDMNMX + 1/2 VIMNMX3 (ALU pipe).  The ALU pipe is the bound (rt 2 per
// SMSP).  The variants move the reduction of the look-ahead (odd) lanes into the
// minimum: min3(min3(best, t, t - p), u, u - p) with t, u and t - p, u - p as plain
// adds (per-feature constants d - p), i.e. ALU work becomes FMA-pipe immediate-form
// adds.  Variant V selects which odd lane pairs take it: 0 none (committed walk),
// 1 all, 2 every other, 3 every third, 4 every fourth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o walk_mix_probe walk_mix_probe.cu
#include <cstdint>
#include <cstdio>

__device__ uint32_t g_sink;

__device__ __forceinline__ uint32_t red(uint32_t t, uint32_t p) { return __viaddmin_u32(t, 0u - p, t); }

template <int K, int V>
__global__ void __launch_bounds__(256) walk_mix(int rounds, uint32_t p, uint32_t seed, long long* cyc) {
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
            best[k] = __vimin3_u32(best[k], ha, hb);
            if (V > 0 && j % V == 0) {
                best[k + 1] = __vimin3_u32(__vimin3_u32(best[k + 1], ha + da, ha + dam), hb + db, hb + dbm);
            } else {
                best[k + 1] = __vimin3_u32(best[k + 1], red(ha + da, p), red(hb + db, p));
            }
            if (k + 2 < K) {
                ha = red(ha + da2, p);
                hb = red(hb + db2, p);
            }
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

template <int K, int V>
void run(int sms, int occ_cap) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk_mix<K, V>, 256, 0);
    if (occ > occ_cap) occ = occ_cap;
    const int blocks = occ * sms;
    long long* cyc;
    cudaMalloc(&cyc, blocks * sizeof(long long));
    const int rounds = 2000;
    walk_mix<K, V><<<blocks, 256>>>(rounds / 10, 67108879u, 1u, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    walk_mix<K, V><<<blocks, 256>>>(rounds, 67108879u, 2u, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    const double visits = (double)blocks * 256 * rounds * K * 2;
    printf("walk_mix K=%2d V=%d occ=%d  %.2f Tvisit/s  %.2f visits/clk/SM\n", K, V, occ,
           visits / (ms * 1e-3) / 1e12, visits / sms / (double)mx);
    delete[] h;
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int rep = 0; rep < 2; ++rep) {
        run<64, 0>(sms, 2);
        run<64, 1>(sms, 2);
        run<64, 2>(sms, 2);
        run<64, 3>(sms, 2);
        run<64, 4>(sms, 2);
        run<32, 0>(sms, 4);
        run<32, 1>(sms, 4);
        run<32, 2>(sms, 4);
    }
    return 0;
}
