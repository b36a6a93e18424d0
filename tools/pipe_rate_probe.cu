// pipe_rate_probe.cu -- issue rate of single integer instruction forms on sm_100a
// (warp-instructions per clock per SMSP), 8 independent chains per thread, 16 warps/SM.
// Which SASS each form becomes is checked with cuobjdump; the walk's costs follow.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rate_probe pipe_rate_probe.cu
#include <cstdint>
#include <cstdio>

__device__ uint32_t g_sink;

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t x, uint32_t a, uint32_t b, uint32_t one) {
    uint32_t r;
    if (OP == 0) {  // add of two vector registers (VIADD / IMAD.IADD / IADD3: ptxas's pick)
        r = x + a;
    } else if (OP == 1) {  // IMAD with three vector registers (opaque multiplier 1)
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(a));
    } else if (OP == 2) {  // VIADDMNMX: min(x + a, b)
        r = min(x + a, b);
    } else if (OP == 3) {  // VIMNMX3
        r = __vimin3_u32(x, a, b);
    } else if (OP == 4) {  // IMAD.HI
        r = __umulhi(x, a);
    } else if (OP == 5) {  // add of a register and an immediate
        r = x + 0x1234567u;
    } else {  // LOP3
        r = (x ^ a) & b;
    }
    return r;
}

template <int OP>
__global__ void __launch_bounds__(256) rate(int iters, uint32_t seed, long long* cyc, uint32_t one) {
    uint32_t v[8], a[8], b[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        v[c] = threadIdx.x * 2654435761u + c * seed;
        a[c] = blockIdx.x * 40503u + 17u * c + seed;
        b[c] = v[c] ^ 0x5bd1e995u;
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = op<OP>(v[c], a[c], b[c], one);
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc ^= v[c];
    if (acc == 0x9e3779b9u) g_sink = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms) {
    const int blocks = 2 * sms;  // 16 warps / SM = 4 per SMSP
    long long* cyc;
    cudaMalloc(&cyc, blocks * sizeof(long long));
    const int iters = 4000;
    rate<OP><<<blocks, 256>>>(iters / 10, 1u, cyc, 1u);
    rate<OP><<<blocks, 256>>>(iters, 2u, cyc, 1u);
    cudaDeviceSynchronize();
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    // warp-instructions per SMSP per clock: 4 warps per SMSP x iters x 128 per iteration
    const double per_smsp = 4.0 * iters * 128 / (double)mx;
    printf("%-28s %.3f warp-instr/clk/SMSP  (rt %.2f)\n", name, per_smsp, 1.0 / per_smsp);
    delete[] h;
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("add reg+reg", sms);
    run<1>("IMAD 3-reg (x*one+a)", sms);
    run<2>("min(x+a, b) VIADDMNMX", sms);
    run<3>("VIMNMX3", sms);
    run<4>("IMAD.HI", sms);
    run<5>("add reg+imm", sms);
    run<6>("LOP3", sms);
    return 0;
}
