// bandhash.cuh -- the LSH band key (include/mhb.h; the reference defines no banding,
// SPEC.md:230, so the definition is this library's and oracle.band_keys restates it).
//
// key(s, band) = splitmix64(h1 << 32 | h2), where over the band's argmin ids x (uint32,
// in row order) two polynomial hashes mod 2^32 run side by side:
//   h1 <- h1 * 0x9E3779B1 + x,   h1_0 = 0x811C9DC5 ^ band
//   h2 <- h2 * 0x85EBCA6B + x,   h2_0 = 0xC2B2AE35 ^ (band * 0x27D4EB2F)
// Each id costs two IMADs on the FMA pipe and nothing on the ALU pipe, so the signing
// kernel (bound by the ALU pipe) can hash its bands in the epilogue almost for free.
#pragma once
#include <cstdint>

namespace mhb {

constexpr uint32_t kBandM1 = 0x9E3779B1u, kBandM2 = 0x85EBCA6Bu;

struct BandHash {
    uint32_t h1, h2;
    __host__ __device__ __forceinline__ explicit BandHash(uint32_t band)
        : h1(0x811C9DC5u ^ band), h2(0xC2B2AE35u ^ (band * 0x27D4EB2Fu)) {}
    __host__ __device__ __forceinline__ void add(uint32_t x) {
        h1 = h1 * kBandM1 + x;
        h2 = h2 * kBandM2 + x;
    }
    __host__ __device__ __forceinline__ unsigned long long key() const {
        unsigned long long z = ((unsigned long long)h1 << 32) | h2;
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
};

}  // namespace mhb
