// doorbell_probe.cu -- host <-> resident-block round trips over mapped host memory.
//
// Measures the building blocks of the per-set doorbell server (csrc/small.cu):
// the poll/acknowledge ping-pong alone, then with input reads over PCIe, output
// writes + fence.sys, in several spellings.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o doorbell_probe doorbell_probe.cu
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>

struct Ctl {
    uint32_t req, done, stop, pad;
};

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// MODE bits: 1 = read n_in u32 inputs (ld.cv) per request, 2 = write n_out u64 outputs
// + fence.sys per request, 4 = poll with ld.relaxed (else ld.acquire), 8 = ack with
// fence.sys + st.volatile (else st.release), 16 = inputs from device memory copy
__device__ unsigned long long g_clk[2];

template <int MODE>
__global__ void server(Ctl* c, const uint32_t* in, int n_in, unsigned long long* out, int n_out) {
    __shared__ uint32_t s_seq;
    __shared__ uint32_t s_acc;
    __shared__ uint32_t xs[4096];
    uint32_t served = 0;
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        if (threadIdx.x == 0) {
            uint32_t s;
            for (;;) {
                s = (MODE & 4) ? ld_relaxed(&c->req) : ld_acq(&c->req);
                if (s != served) break;
            }
            s_seq = s;
            s_acc = 0;
        }
        __syncthreads();
        const uint32_t seq = s_seq;
        if (seq == 0xffffffffu) {
            if (threadIdx.x == 0) {
                unsigned long long t1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                g_clk[0] = clock64() - c0;
                g_clk[1] = t1 - t0;
            }
            return;
        }
        uint32_t acc = 0;
        if (MODE & 64) {
            const uint4* in4 = reinterpret_cast<const uint4*>(in);
            for (int k = threadIdx.x; k < n_in / 4; k += blockDim.x) {
                const uint4 v = __ldcv(in4 + k);
                acc += v.x + v.y + v.z + v.w;
            }
        } else if (MODE & 1) {
            for (int k = threadIdx.x; k < n_in; k += blockDim.x) acc += __ldcv(in + k);
        }
        if (acc) atomicAdd(&s_acc, acc);
        __syncthreads();
        if (MODE & 128) {  // the per-set compute: 128 hashes x min(n_in, 4096) ids, Shoup lanes
            const int n = n_in < 4096 ? n_in : 4096;
            for (int k = threadIdx.x; k < n; k += blockDim.x) xs[k] = (uint32_t)k * 2654435761u % 1048583u;
            __syncthreads();
            if (threadIdx.x < 128) {
                const uint32_t p = 1048583u, a = 1000u + threadIdx.x + seq, b = 77u * threadIdx.x;
                const uint32_t ap = (uint32_t)(((unsigned long long)a << 32) / p);
                uint32_t best = 0xffffffffu, arg = 0;
                for (int k = 0; k < n; ++k) {
                    const uint32_t x = xs[k];
                    uint32_t r = a * x - __umulhi(ap, x) * p;
                    r = min(r, r - p);
                    r = min(r + b, r + b - p);
                    if (r < best) { best = r; arg = x; }
                }
                if (arg == 0xdeadbeefu) atomicAdd(&s_acc, 1u);
            }
            __syncthreads();
        }
        if (MODE & 2) {
            for (int k = threadIdx.x; k < n_out; k += blockDim.x) out[k] = (unsigned long long)seq * 1000 + k + s_acc;
            if (!(MODE & 32)) __threadfence_system();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (MODE & 8) {
                __threadfence_system();
                st_vol(&c->done, seq);
            } else {
                st_rel(&c->done, seq);
            }
        }
        served = seq;
    }
}

template <int MODE>
void run(const char* name, int n_in, int n_out) {
    Ctl* c;
    uint32_t* in;
    unsigned long long* out;
    cudaHostAlloc((void**)&c, sizeof(Ctl), cudaHostAllocMapped);
    cudaHostAlloc((void**)&in, 65536 * 4, cudaHostAllocMapped);
    cudaHostAlloc((void**)&out, 65536 * 8, cudaHostAllocMapped);
    memset(c, 0, sizeof(Ctl));
    for (int i = 0; i < 65536; ++i) in[i] = i;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    server<MODE><<<1, 256, 0, st>>>(c, in, n_in, out, n_out);
    const int iters = 20000;
    double t_best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < iters; ++i) {
            const uint32_t seq = rep * iters + i + 1;
            __atomic_store_n(&c->req, seq, __ATOMIC_RELEASE);
            while (__atomic_load_n(&c->done, __ATOMIC_ACQUIRE) != seq) __builtin_ia32_pause();
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
        if (us < t_best) t_best = us;
    }
    __atomic_store_n(&c->req, 0xffffffffu, __ATOMIC_RELEASE);
    cudaStreamSynchronize(st);
    unsigned long long clk[2];
    cudaMemcpyFromSymbol(clk, g_clk, sizeof clk);
    printf("%-40s in=%5d u32 out=%5d u64  %.2f us/round trip  (SM clock %.0f MHz)\n", name, n_in, n_out, t_best,
           clk[1] ? clk[0] * 1e3 / clk[1] : 0.0);
    cudaStreamDestroy(st);
    cudaFreeHost(c);
    cudaFreeHost(in);
    cudaFreeHost(out);
}

// Launch-per-request baseline: kernel reading/writing mapped memory + stream sync.
__global__ void once(const uint32_t* in, int n_in, unsigned long long* out, int n_out) {
    uint32_t acc = 0;
    for (int k = threadIdx.x; k < n_in; k += blockDim.x) acc += in[k];
    for (int k = threadIdx.x; k < n_out; k += blockDim.x) out[k] = k + acc;
}

void run_launch(int n_in, int n_out) {
    uint32_t* in;
    unsigned long long* out;
    cudaHostAlloc((void**)&in, 65536 * 4, cudaHostAllocMapped);
    cudaHostAlloc((void**)&out, 65536 * 8, cudaHostAllocMapped);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    const int iters = 5000;
    double t_best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < iters; ++i) {
            once<<<1, 256, 0, st>>>(in, n_in, out, n_out);
            cudaStreamSynchronize(st);
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
        if (us < t_best) t_best = us;
    }
    printf("%-40s in=%5d u32 out=%5d u64  %.2f us/call\n", "launch + stream sync", n_in, n_out, t_best);
    cudaStreamDestroy(st);
    cudaFreeHost(in);
    cudaFreeHost(out);
}

int main() {
    cudaFree(0);
    run<0>("ping-pong acquire/release", 0, 0);
    run<4>("ping-pong relaxed/release", 0, 0);
    run<8>("ping-pong acquire/fence+volatile", 0, 0);
    run<12>("ping-pong relaxed/fence+volatile", 0, 0);
    run<1>("+ inputs", 64, 0);
    run<1>("+ inputs", 2048, 0);
    run<2>("+ outputs", 0, 128);
    run<2>("+ outputs", 0, 2048);
    run<3>("+ inputs + outputs", 64, 128);
    run<7>("+ inputs + outputs (relaxed poll)", 64, 128);
    run<15>("+ inputs + outputs (relaxed, fence+vol)", 64, 128);
    run<1 + 2 + 32>("in + out, fence by thread 0 only", 64, 128);
    run<64 + 2>("in v4 + out", 64, 128);
    run<64 + 2 + 32>("in v4 + out, fence by thread 0 only", 64, 128);
    run<64 + 2 + 32>("in v4 + out, fence by thread 0 only", 1024, 128);
    run<64 + 2 + 32>("in v4 + out, fence by thread 0 only", 4096, 128);
    run<64 + 2 + 32>("in v4 + out, fence by thread 0 only", 16384, 2048);
    run<64 + 2 + 32 + 128>("in v4 + compute 128x50 + out", 64, 128);
    run<64 + 2 + 32 + 128>("in v4 + compute 128x200 + out", 200, 128);
    run_launch(0, 0);
    run_launch(64, 128);
    return 0;
}
