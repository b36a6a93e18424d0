// sign_internal.h -- structures shared by the signature kernels and the host pipeline.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace mhb {

enum { KIND_ITERATIVE = 0, KIND_RANDOM = 1 };

constexpr int kChunk = 1024;         // largest virtual set (SignArgs::chunk <= kChunk); longer sets are split
constexpr int kBlock = 256;          // threads per CTA of the main kernel
constexpr int kEpiSmemLanes = 2048;  // epilogue table staged in shared memory up to this many lanes

// Per hash lane i: h_i(x) = (A*x + B) mod p, Ap = floor(A*2^32/p) (Shoup companion).
struct LaneTab {
    uint32_t A, Ap, B, pad;
};
// Per hash lane i, for the argmin recovery x = (h - B) * inv mod p:
// B (the lane offset), inv = A^{-1} mod p and its Shoup companion.
struct InvTab {
    uint32_t B, inv, invp, pad;
};
// A virtual set: up to kChunk consecutive features of one set.
//   f0   : index of its first feature in ids
//   meta : set << 12 | merge << 11 | (n - 1); merge = the set has several chunks
struct VSet {
    long long f0;
    long long meta;
};
struct Sched {
    unsigned long long next;     // dynamic counter over work items (group, lane pass)
    unsigned long long n_vsets;  // virtual sets planned
    unsigned long long n_big;    // sets in merge mode (finalize list)
    unsigned long long done;     // CTAs finished (STATIC kernels: the last one finalizes)
    int32_t status;              // small batches: the call's status word, copied out by the last CTA
    int32_t pad2;
};

struct Geometry {
    int K;         // hash lanes per thread
    int G;         // lane groups per warp
    int F;         // sets per warp group (one per slice; G*F = 32)
    int log2F;
    int n_super;   // lane passes per set (n_hash > 32*K)
    int L;         // lanes per pass = G*K
    int64_t n_tot; // padded lane count = n_super*L
};

struct WorkspaceLayout {
    size_t sched, hist, tab, inv, big, vsets, total;
};

struct SignArgs {
    const int64_t* indptr;
    const uint32_t* ids;
    int64_t n_sets;
    uint32_t p;
    uint32_t b;
    uint64_t ia;
    int32_t n_hash;
    int32_t F, log2F, n_super, L, K;
    int64_t n_tot;
    int32_t kind;
    LaneTab* tab;
    InvTab* inv;
    Sched* sched;
    unsigned* hist;   // [2*kChunk]: virtual-set size histogram, then scatter cursors (plan kernels);
                      // in a STATIC sign kernel's copy: the caller's status word, or null
    int64_t* big;
    VSet* vsets;
    int32_t* status;
    void* out;
    const uint32_t* ra;
    const uint32_t* rb;
    // fused LSH band keys (mhb_sign_iterative_csr_bands); keys == nullptr: off
    unsigned long long* keys;
    int32_t rows;       // rows per band (divides K and n_hash)
    int32_t write_sig;  // 0: keys only (out still serves long-set rows as scratch)
    int32_t fpq;        // random family, p <= 2^23: lane tables hold rd(w/p) and the folded offset
    int32_t chunk;      // features per virtual set of this launch (256, 512 or 1024: choose_chunk);
                        // appended last so the main kernels' parameter layout is unchanged
};

// K = 0: the default lanes per thread for n_hash (large batches); K in {8,16,32,64}
// forces it (small batches take a smaller K so the grid fills the SMs: pick_lanes).
Geometry choose_geometry(int kind, int32_t n_hash, int K = 0);

// 64-bit-residue path for primes 2^31 <= p < 2^63 (wide.cu).
int launch_sign_wide(bool iter, const int64_t* indptr, const uint32_t* ids, int64_t n_sets, uint64_t a, uint64_t b,
                     const uint64_t* ra, const uint64_t* rb, uint64_t prime, int32_t n_hash, void* out,
                     int32_t out_dtype, int32_t* status, cudaStream_t st);
WorkspaceLayout workspace_layout(int64_t n_sets, int64_t nnz, int32_t n_hash);
// Virtual-set size for a batch (a function of its shape alone, so the workspace size and
// the launch agree).
int choose_chunk(int64_t n_sets, int64_t nnz, int32_t n_hash);

// Host-side parameter checks shared by every signing entry (errors as in launch_sign).
int check_sign_params(int kind, uint64_t a, uint64_t b, bool have_random_arrays, uint64_t prime, int32_t n_hash);

int launch_sign(int kind, const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t nnz,
                uint64_t a, uint64_t b, const uint32_t* ra, const uint32_t* rb, uint64_t prime,
                int32_t n_hash, void* out, int32_t out_dtype, int32_t* status, void* workspace,
                size_t workspace_bytes, cudaStream_t st, unsigned long long* keys = nullptr,
                int32_t rows_per_band = 0, int32_t write_sig = 1);

// Output-sensitive iterative-family kernel (gap.cu): enumerates, per feature, only the
// lanes whose hash falls below the set's threshold.  `gap_preferred` is the cost model
// (MHB_GAP=0/1 forces it off/on); launch_sign_gap needs the lane tables of plan_count_kernel
// and a zeroed Sched::next.
struct DeviceInfo;
bool gap_preferred(int kind, uint64_t prime, int32_t n_hash, int64_t n_sets, int64_t nnz);
// Sets that make one full wave of the enumerating kernel's tiles on a B200 (4 CTAs x 148 SMs).
int64_t gap_full_wave_sets(int32_t n_hash, int64_t n_sets, int64_t nnz);
int launch_sign_gap(const SignArgs& S, int64_t nnz, int32_t out_dtype, const DeviceInfo& dev, cudaStream_t st);

}  // namespace mhb
