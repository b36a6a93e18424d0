// modarith.cuh -- exact u32 modular arithmetic for primes p < 2^31 on sm_100a.
//
// Every hash value lives in [0, p).  The reference computes the same residues
// with int64 '%' (kernels.py:33,36,64-65); here each reduction is one
// conditional subtract expressed as an unsigned min, which ptxas lowers to a
// single DPX instruction: min(t, t - p) == VIADDMNMX.U32 t, -p, t.
#pragma once
#include <cstdint>

namespace mhb {

// t in [0, 2p) -> t mod p.  (t - p wraps to >= 2^32 - p when t < p.)
__device__ __forceinline__ uint32_t reduce_once(uint32_t t, uint32_t p) {
    return __viaddmin_u32(t, 0u - p, t);
}

// Shoup multiply: w < p < 2^31, wp = floor(w * 2^32 / p), any x < 2^32.
// Returns w*x mod p, partially reduced into [0, 2p).
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t w, uint32_t wp, uint32_t x, uint32_t p) {
    uint32_t q = __umulhi(wp, x);
    return w * x - q * p;
}

// (w*x + c) mod p for w, c < p < 2^31: fully reduced, safe for every p < 2^31.
__device__ __forceinline__ uint32_t mul_add_mod(uint32_t w, uint32_t wp, uint32_t c,
                                                uint32_t x, uint32_t p) {
    uint32_t r = reduce_once(shoup_lazy(w, wp, x, p), p);
    return reduce_once(r + c, p);
}

// (w*x + c) mod p with the add folded before reduction: needs 3p < 2^32.
// One instruction shorter than mul_add_mod; used on the random family's per-visit path.
__device__ __forceinline__ uint32_t mul_add_mod_narrow(uint32_t w, uint32_t wp, uint32_t c,
                                                       uint32_t x, uint32_t p) {
    uint32_t q = __umulhi(wp, x);
    uint32_t r = w * x + c - q * p;          // in [0, 3p)
    r = reduce_once(r, p);
    return reduce_once(r, p);
}

// (w*x + c) mod p with one ALU instruction, needs 3p < 2^32: r = w*x + c - q*p lies in
// [0, 3p); the two subtractions run on the FMA pipe and a single 3-way unsigned min
// (VIMNMX3) picks the residue (the wrapped candidates are >= 2^32 - 2p).
__device__ __forceinline__ uint32_t mul_add_mod_min3(uint32_t w, uint32_t wp, uint32_t c,
                                                     uint32_t x, uint32_t p) {
    uint32_t q = __umulhi(wp, x);
    uint32_t r = w * x + c - q * p;
    return __vimin3_u32(r, r - p, r - 2u * p);
}

// Variants taking negp = 2^32 - p from an opaque (kernel-parameter) register:
// r = w*x + c + q*negp is one IMAD per term, where the "- q*p" spelling costs an
// extra negation of q (IMAD.MOV/IADD3) on the per-visit path.
__device__ __forceinline__ uint32_t mul_add_mod_narrow_n(uint32_t w, uint32_t wp, uint32_t c, uint32_t x,
                                                         uint32_t p, uint32_t negp) {
    const uint32_t q = __umulhi(wp, x);
    const uint32_t r = w * x + c + q * negp;  // in [0, 3p)
    return reduce_once(reduce_once(r, p), p);
}
__device__ __forceinline__ uint32_t mul_add_mod_n(uint32_t w, uint32_t wp, uint32_t c, uint32_t x, uint32_t p,
                                                  uint32_t negp) {
    const uint32_t q = __umulhi(wp, x);
    const uint32_t r = reduce_once(w * x + q * negp, p);
    return reduce_once(r + c, p);
}
__device__ __forceinline__ uint32_t mul_add_mod_min3_n(uint32_t w, uint32_t wp, uint32_t c, uint32_t x, uint32_t p,
                                                       uint32_t negp) {
    const uint32_t q = __umulhi(wp, x);
    const uint32_t r = w * x + c + q * negp;
    return __vimin3_u32(r, r + negp, r + 2u * negp);
}

// Host/device helpers on 64-bit integers (setup only, never per visit).
__host__ __device__ __forceinline__ uint32_t shoup_companion(uint32_t w, uint32_t p) {
    return (uint32_t)(((uint64_t)w << 32) / p);
}

// Modular inverse of w in Z_p (w != 0 mod p, p prime) by the extended Euclid.  The
// remainders stay below 2^32, so the quotients are 32-bit divisions (the 64-bit
// division the naive spelling emits is a long emulated sequence on the GPU); the
// Bezout coefficients are bounded by p in magnitude.
__host__ __device__ inline uint32_t inv_mod(uint32_t w, uint32_t p) {
    int64_t t = 0, nt = 1;
    uint32_t r = p, nr = w % p;
    while (nr != 0) {
        const uint32_t q = r / nr;
        const int64_t tmp = t - (int64_t)q * nt;
        t = nt;
        nt = tmp;
        const uint32_t rr = r - q * nr;
        r = nr;
        nr = rr;
    }
    if (t < 0) t += p;
    return (uint32_t)t;
}

}  // namespace mhb
