// common.cu -- error state, primality test, device-property cache.
#include "common.h"

#include <mutex>
#include <string>

namespace mhb {

static thread_local char g_err[512] = {0};

int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

void clear_error() { g_err[0] = 0; }

static uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)((unsigned __int128)a * b % m);
}

static uint64_t powmod64(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod64(r, b, m);
        b = mulmod64(b, b, m);
        e >>= 1;
    }
    return r;
}

static bool is_prime_u64_uncached(uint64_t n);

// Deterministic Miller-Rabin (the 12 bases are exact below 3.3e24).  A per-thread memo of
// the last few primes confirmed: every signing call checks its modulus (~1.6 us of
// 128-bit modular arithmetic, a tenth of a per-set call), and callers reuse one family.
bool is_prime_u64(uint64_t n) {
    static thread_local uint64_t memo[4] = {0, 0, 0, 0};
    static thread_local unsigned next = 0;
    for (uint64_t m : memo)
        if (m == n && n != 0) return true;
    if (!is_prime_u64_uncached(n)) return false;
    memo[next++ & 3] = n;
    return true;
}

static bool is_prime_u64_uncached(uint64_t n) {
    static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t b : bases) {
        if (n % b == 0) return n == b;
    }
    uint64_t d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; ++r; }
    for (uint64_t b : bases) {
        uint64_t x = powmod64(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int i = 1; i < r; ++i) {
            x = mulmod64(x, x, n);
            if (x == n - 1) { composite = false; break; }
        }
        if (composite) return false;
    }
    return true;
}

int current_device_info(DeviceInfo* out) {
    static std::mutex mu;
    static DeviceInfo cache[64];
    static bool have[64] = {false};
    int dev = 0;
    int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    if (dev < 0 || dev >= 64) return set_error(MHB_ERR_CUDA, "device index %d out of range", dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!have[dev]) {
        DeviceInfo d{dev, 0, 0};
        int v = 0;
        rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev), "sm count");
        if (rc) return rc;
        d.sms = v;
        rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
                        "smem optin");
        if (rc) return rc;
        d.smem_optin = (size_t)v;
        cache[dev] = d;
        have[dev] = true;
    }
    *out = cache[dev];
    return MHB_OK;
}

}  // namespace mhb

extern "C" const char* mhb_last_error(void) { return mhb::g_err; }

extern "C" const char* mhb_version(void) {
    return "mhb 0.1.0 (sm_100a; iterative + random MinHash over CSR)";
}
