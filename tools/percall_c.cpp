// percall_c.cpp -- per-call latency of mhb_sign_csr_host for one small set, from C
// (no Python / ctypes in the loop): the per-set reference call shape (N=128, ~50 ids).
// usage: percall_c [ids] [hashes] [out_dtype 0=u32 1=i64] [pinned 0/1]
// Build (from tools/): g++ -O2 -I../include -I/usr/local/cuda/include percall_c.cpp \
//   -L../paper_1401_6124_b200/lib -lmhb -L/usr/local/cuda/lib64 -lcudart \
//   -Wl,-rpath,'$ORIGIN/../paper_1401_6124_b200/lib' -o percall_c
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mhb.h"

#include <cuda_runtime.h>

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 50, n_hash = argc > 2 ? atoi(argv[2]) : 128;
    const int out_dtype = argc > 3 ? atoi(argv[3]) : MHB_OUT_I64;  // 0 u32, 1 i64
    const bool pinned = argc > 4 && atoi(argv[4]);
    const uint32_t p = 1048583u;
    std::vector<uint32_t> ids(n);
    for (int k = 0; k < n; ++k) ids[k] = (uint32_t)((k * 2654435761ull) % p);
    int64_t indptr[2] = {0, n};
    std::vector<long long> out_vec(n_hash);
    long long* out = out_vec.data();
    if (pinned) cudaMallocHost((void**)&out, (size_t)n_hash * 8);
    int32_t st = 0;
    for (int i = 0; i < 200; ++i)
        if (mhb_sign_csr_host(0, indptr, ids.data(), 1, n, 12345, 678, nullptr, nullptr, p, n_hash, out,
                              out_dtype, &st, 0)) {
            printf("error: %s\n", mhb_last_error());
            return 1;
        }
    double best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        const int iters = n_hash > 10000 ? 300 : 5000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < iters; ++i)
            mhb_sign_csr_host(0, indptr, ids.data(), 1, n, 12345 + (i & 7), 678, nullptr, nullptr, p, n_hash,
                              out, out_dtype, &st, 0);
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
        best = us < best ? us : best;
    }
    printf("mhb_sign_csr_host from C: %d ids x %d hashes, %s out, %s: %.2f us/call\n", n, n_hash,
           out_dtype == MHB_OUT_I64 ? "int64" : "uint32", pinned ? "pinned" : "pageable", best);
    mhb_host_release();
    return 0;
}
