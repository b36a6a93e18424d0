// atoms_probe.cu -- shared-memory atomic throughput on the B200 (for the histogram design).
// Each thread issues `iters` red.shared.add.u32 to addresses of a chosen pattern; reports
// lanes/clk/SM.  Patterns: 0 = lane's own bank (word i*32 + lane), 1 = 2-way (lanes L and
// L+16 share bank set), 2 = random word in a 4096-word table, 3 = same as 0 with 16 active
// lanes, 4 = plain LDS+IADD+STS on the lane's own bank (non-atomic RMW), 5 = atom with return.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_probe atoms_probe.cu
#include <cstdint>
#include <cstdio>

__device__ uint32_t g_sink;

template <int PAT>
__global__ void __launch_bounds__(512) probe(int iters, uint32_t seed, int words) {
    extern __shared__ uint32_t t[];
    for (int i = threadIdx.x; i < words; i += blockDim.x) t[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(t);
    uint32_t h = seed * 2654435761u + threadIdx.x * 40503u + blockIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            h = h * 1664525u + 1013904223u;
            uint32_t w;
            if (PAT == 0 || PAT == 3 || PAT == 4 || PAT == 5) w = ((h >> 20) & 127) * 32 + lane;
            else if (PAT == 1) w = ((h >> 20) & 255) * 16 + (lane & 15);
            else w = (h >> 20) & 4095;
            const uint32_t a = base + w * 4;
            if (PAT == 3 && lane >= 16) continue;
            if (PAT == 4) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v + 1));
            } else if (PAT == 5) {
                uint32_t o;
                asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(o) : "r"(a));
                acc += o;
            } else {
                asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a));
            }
        }
    }
    __syncthreads();
    if (acc == 0x12345678u) g_sink = acc;
    if (threadIdx.x == 0 && t[0] == 0x12345678u) g_sink = t[1];
}

template <int PAT>
void run(const char* name, int threads, int sms) {
    const int words = 4096;
    const size_t smem = words * 4;
    int occ = 0;
    cudaFuncSetAttribute(probe<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<PAT>, threads, smem);
    const int blocks = occ * sms;
    const int iters = 4096;
    probe<PAT><<<blocks, threads, smem>>>(iters / 10, 1, words);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<PAT><<<blocks, threads, smem>>>(iters, 2, words);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8 * (PAT == 3 ? 0.5 : 1.0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s threads=%d occ=%d  %.3f Tops/s  %.2f lanes/clk/SM (at %d MHz)\n", name, threads, occ,
           ops / (ms * 1e-3) / 1e12, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int th : {256, 512, 1024}) {
        run<0>("red own bank", th, sms);
        run<1>("red 2-way (16 replicas)", th, sms);
        run<2>("red random 4096", th, sms);
        run<3>("red own bank, 16 lanes", th, sms);
        run<4>("lds+sts own bank", th, sms);
        run<5>("atom(ret) own bank", th, sms);
    }
    return 0;
}
