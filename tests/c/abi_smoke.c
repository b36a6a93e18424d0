/*
 * abi_smoke.c -- a plain C consumer of include/mhb.h (no Python, no torch): the
 * binding a C/C++/cgo/JNI caller would write.  Signs the reference's known-answer
 * set {2, 5} under IterativeFamily(a=3, b=5, p=7, N=1) -> [5]
 * (tests/test_minhash.py:90-94) and a singleton under N=16 -> all 42, through both
 * the device entry and the host-buffer pipeline.
 *
 * build: gcc -O2 abi_smoke.c -I../../include -I/usr/local/cuda/include \
 *            -L../../paper_1401_6124_b200/lib -lmhb -L/usr/local/cuda/lib64 -lcudart
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "mhb.h"

static int fail(const char* what) {
    fprintf(stderr, "FAIL %s: %s\n", what, mhb_last_error());
    return 1;
}

int main(void) {
    /* host pipeline: {2,5}, a=3, b=5, p=7, N=1 -> [5] */
    int64_t indptr[2] = {0, 2};
    uint32_t ids[2] = {2, 5};
    int64_t out64[1] = {-1};
    int32_t status = -1;
    if (mhb_sign_csr_host(0, indptr, ids, 1, 2, 3, 5, NULL, NULL, 7, 1, out64, MHB_OUT_I64, &status, 0))
        return fail("mhb_sign_csr_host");
    if (out64[0] != 5 || status != 0) {
        fprintf(stderr, "FAIL known answer: got %lld status %d\n", (long long)out64[0], status);
        return 1;
    }

    /* device entry: singleton {42}, N=16, p=7757 -> all 42 */
    int64_t h_ip[2] = {0, 1};
    uint32_t h_ids[1] = {42};
    int64_t* d_ip;
    uint32_t* d_ids;
    uint32_t* d_out;
    int32_t* d_status;
    void* d_ws;
    const size_t ws = mhb_sign_workspace_bytes(1, 1, 16);
    cudaMalloc((void**)&d_ip, sizeof h_ip);
    cudaMalloc((void**)&d_ids, sizeof h_ids);
    cudaMalloc((void**)&d_out, 16 * sizeof(uint32_t));
    cudaMalloc((void**)&d_status, sizeof(int32_t));
    cudaMalloc(&d_ws, ws);
    cudaMemcpy(d_ip, h_ip, sizeof h_ip, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ids, h_ids, sizeof h_ids, cudaMemcpyHostToDevice);
    if (mhb_sign_iterative_csr(d_ip, d_ids, 1, 1, 1234, 99, 7757, 16, d_out, MHB_OUT_U32, d_status, d_ws, ws, NULL))
        return fail("mhb_sign_iterative_csr");
    uint32_t h_out[16];
    cudaMemcpy(h_out, d_out, sizeof h_out, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 16; ++i)
        if (h_out[i] != 42) {
            fprintf(stderr, "FAIL singleton lane %d: %u\n", i, h_out[i]);
            return 1;
        }
    /* argument errors come back before any launch, with text */
    if (mhb_sign_iterative_csr(d_ip, d_ids, 1, 1, 1234, 99, 7758, 16, d_out, MHB_OUT_U32, d_status, d_ws, ws, NULL) !=
        MHB_ERR_INVALID)
        return fail("non-prime modulus not rejected");
    printf("abi_smoke ok (%s)\n", mhb_version());
    mhb_host_release();
    return 0;
}
