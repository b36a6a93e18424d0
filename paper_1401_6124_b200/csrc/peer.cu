// peer.cu -- peer-memory gather target for fused sign + gather.
//
// The only collective of the row-sharded path is the gather of signature blocks to
// one rank.  Instead of signing into a local block and then running a gather, every
// rank maps the destination rank's output matrix (CUDA IPC; an NVLink peer mapping
// when the ranks sit on different GPUs) and launches the signing kernels with `out`
// pointing at its own rows of that matrix: the epilogue's 16-byte stores (and the
// long-set red.global.min merges) travel to the destination as each tile finishes,
// overlapping the transfer with the remaining compute.  No kernel changes: the
// signing kernels only ever see an `out` pointer.
#include <cuda_runtime.h>

#include <cstring>

#include "common.h"

using namespace mhb;

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");

extern "C" int mhb_peer_alloc(size_t bytes, int32_t device, void** ptr, unsigned char* handle) {
    clear_error();
    if (!ptr || !handle) return set_error(MHB_ERR_INVALID, "ptr and handle are required");
    *ptr = nullptr;
    int rc = cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (rc) return rc;
    void* p = nullptr;
    rc = cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc(peer buffer)");
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    rc = cuda_check(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
    if (rc) {
        cudaFree(p);
        return rc;
    }
    std::memcpy(handle, &h, sizeof(h));
    *ptr = p;
    return MHB_OK;
}

extern "C" int mhb_peer_open(const unsigned char* handle, int32_t device, void** ptr) {
    clear_error();
    if (!ptr || !handle) return set_error(MHB_ERR_INVALID, "ptr and handle are required");
    *ptr = nullptr;
    int rc = cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return cuda_check(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

extern "C" int mhb_peer_close(void* ptr) {
    clear_error();
    return cuda_check(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

extern "C" int mhb_peer_free(void* ptr) {
    clear_error();
    return cuda_check(cudaFree(ptr), "cudaFree(peer buffer)");
}
