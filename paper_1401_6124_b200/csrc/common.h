// common.h -- host-side helpers shared by the libmhb translation units:
// thread-local error text, CUDA error mapping, primality, device properties.
#pragma once
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include "mhb.h"

namespace mhb {

int set_error(int code, const char* fmt, ...);
void clear_error();

inline int cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return MHB_OK;
    return set_error(MHB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Deterministic Miller-Rabin for 64-bit n (same witness set as the reference,
// modmath.py:11-47).
bool is_prime_u64(uint64_t n);

struct DeviceInfo {
    int device;
    int sms;
    size_t smem_optin;
};
int current_device_info(DeviceInfo* out);

}  // namespace mhb
