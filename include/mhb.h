/*
 * mhb.h -- C ABI of libmhb, the B200 (sm_100a) MinHash signature library.
 *
 * This is the drop-in boundary for the reference's compiled hot loops
 * (arXiv 1401.6124 reference package `minhashlab`):
 *
 *   reference (numba, one set per call)                 this ABI (CUDA, CSR batch per call)
 *   -------------------------------------------------   ---------------------------------------
 *   kernels.sign_iterative(ids, a, b, p, n)             mhb_sign_iterative_csr
 *       /root/reference/pkg/src/minhashlab/kernels.py:44-73
 *   kernels.sign_random(ids, a, b, p)                   mhb_sign_random_csr
 *       /root/reference/pkg/src/minhashlab/kernels.py:21-41
 *   minhash.signature(s, family) dispatch               (Python host layer, calls the two above)
 *       /root/reference/pkg/src/minhashlab/minhash.py:91-110
 *   minhash.estimate_jaccard(g1, g2)                    mhb_jaccard_pairs / mhb_jaccard_block
 *       /root/reference/pkg/src/minhashlab/minhash.py:130-137, bench.py:165-168
 *   stats.bucket_uniformity_experiment counts           mhb_bucket_hist_iterative / _random
 *       /root/reference/pkg/src/minhashlab/stats.py:221-224 (eval_all(x) % buckets, bincount)
 *
 * Output semantics are the reference's: out[s*n_hash + i] is the feature id of
 * set s that minimises h_i over the set (argmin, not the min hash value), with
 * h_i(x) = ((a+i)*x + i*b) mod p (iterative, families.py:124-131) or
 * h_i(x) = (a_i*x + b_i) mod p (random, families.py:70-112).  Every member is a
 * bijection on [0,p), so the reference's "smallest id wins ties" rule
 * (minhash.py:94-96) never decides a result and the argmin is unique.
 *
 * Conventions
 *  - All array pointers passed to mhb_sign_* / mhb_jaccard_* / mhb_bucket_hist_*
 *    are DEVICE pointers owned by the caller.  The library allocates nothing on
 *    these paths; scratch comes from the caller's workspace.
 *  - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t, or
 *    NULL for the legacy default stream).  No host synchronisation happens inside.
 *  - CSR: indptr is int64[n_sets+1] (indptr[0] need not be 0: ids are addressed
 *    as ids[indptr[s] .. indptr[s+1])), ids is uint32[>= indptr[n_sets]] and all of
 *    ids[0 .. indptr[n_sets]) must be readable (idle warp lanes read ids[0]).
 *    Ids may be in any order and may repeat inside a set (min is idempotent).
 *  - Data errors found on the device are OR-ed into *status (reset to 0 by the
 *    call): MHB_STATUS_EMPTY_SET mirrors minhash.py:97-98, MHB_STATUS_ID_GE_PRIME
 *    mirrors minhash.py:99-101.  Rows with a flagged error hold unspecified ids.
 *  - Return value: MHB_OK or an MHB_ERR_* code; mhb_last_error() gives the text
 *    (thread-local).  Argument errors are detected before any launch.
 *  - Supported modulus: 3 <= prime < 2^63, prime must be prime.  Primes < 2^31 (every
 *    BASELINE configuration: the largest is 1,073,741,827) run the tuned u32 kernels;
 *    2^31 <= p < 2^63 runs a correctness-first 64-bit path (wide.cu), the analogue of
 *    the reference's int64 / exact fallback paths (minhash.py:102-127).
 */
#ifndef MHB_H_
#define MHB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mhb_error {
    MHB_OK = 0,
    MHB_ERR_INVALID = 1,     /* bad argument (maps to the reference's ValueError) */
    MHB_ERR_CUDA = 2,        /* CUDA runtime error */
    MHB_ERR_UNSUPPORTED = 3  /* valid for the reference, outside this library's range */
};

enum mhb_out_dtype {
    MHB_OUT_U32 = 0,         /* uint32 argmin ids (compact; ids < prime < 2^31) */
    MHB_OUT_I64 = 1          /* int64 argmin ids (the reference's dtype, kernels.py:29,51-52) */
};

enum mhb_status_bits {
    MHB_STATUS_EMPTY_SET = 1,    /* some row has indptr[s+1] <= indptr[s] */
    MHB_STATUS_ID_GE_PRIME = 2,  /* some feature id >= prime */
    MHB_STATUS_BAD_PARAM = 4     /* random family: some a_i not in [1,p) or b_i not in [0,p) */
};

/* Library identification. */
const char* mhb_version(void);

/* Text of the last error raised on the calling thread ("" if none). */
const char* mhb_last_error(void);

/* Scratch bytes mhb_sign_* needs for this problem shape (same for both families).
 * Monotone in n_sets and nnz: a workspace sized for the largest batch of a given n_hash
 * serves every smaller one. */
size_t mhb_sign_workspace_bytes(int64_t n_sets, int64_t nnz, int32_t n_hash);

/* Which kernel mhb_sign_iterative_csr runs for this batch shape (a report for benchmarks
 * and profiles; results are identical either way):
 *   0  visiting kernel: every (feature, hash) pair, 2.5 instructions per visit
 *      (sign_kernel / sign_small_batch_kernel, csrc/sign.cu);
 *   1  enumerating kernel: per feature only the hashes under the set's threshold, found
 *      through the three-gap structure of the iterative family's arithmetic progression
 *      (sign_gap_kernel, csrc/gap.cu; kernels.py:62-72 is the progression it exploits).
 * The choice is a cost model over (n_hash, mean set size); batches of <= 16,384 sets take
 * kernel 1 only from a full wave of its tiles up (3,552 sets at n_hash 2048).  MHB_GAP=0/1
 * forces it where it is supported (prime < 2^31, n_hash <= 26,624). */
int32_t mhb_sign_iterative_path(int64_t n_sets, int64_t nnz, uint64_t prime, int32_t n_hash);

/*
 * Iterative family signatures (replaces kernels.sign_iterative, kernels.py:44-73,
 * for a whole CSR batch).  a, b are the family base parameters
 * (IterativeFamily.base.a / .base.b, families.py:133-147), with a + n_hash < prime.
 * out: n_sets * n_hash entries of out_dtype, row-major.
 */
int mhb_sign_iterative_csr(const int64_t* indptr, const uint32_t* ids,
                           int64_t n_sets, int64_t nnz,
                           uint64_t a, uint64_t b, uint64_t prime, int32_t n_hash,
                           void* out, int32_t out_dtype, int32_t* status,
                           void* workspace, size_t workspace_bytes, void* stream);

/*
 * Random (Carter-Wegman) family signatures (replaces kernels.sign_random,
 * kernels.py:21-41).  a, b: device uint32[n_hash] (RandomFamily.a / .b,
 * families.py:193-204), 1 <= a_i < prime, 0 <= b_i < prime.
 */
int mhb_sign_random_csr(const int64_t* indptr, const uint32_t* ids,
                        int64_t n_sets, int64_t nnz,
                        const uint32_t* a, const uint32_t* b, uint64_t prime, int32_t n_hash,
                        void* out, int32_t out_dtype, int32_t* status,
                        void* workspace, size_t workspace_bytes, void* stream);

/*
 * Iterative signatures with the LSH band keys of mhb_band_keys computed in the
 * signing epilogue (no re-read of the signature matrix).  keys: device uint64
 * [n_sets * n_hash/rows_per_band].  write_signatures = 0 skips storing the
 * signatures (out is still required, all n_sets * n_hash entries: long sets use their
 * rows as merge scratch, and batches signed by the enumerating kernel -- see
 * mhb_sign_iterative_path -- store the rows and hash the keys from them).
 * Needs the K = 32/64 lane geometry (n_hash >= 32), rows_per_band a multiple of 4
 * dividing both K and n_hash, and prime < 2^31; else MHB_ERR_UNSUPPORTED.
 */
int mhb_sign_iterative_csr_bands(const int64_t* indptr, const uint32_t* ids,
                                 int64_t n_sets, int64_t nnz,
                                 uint64_t a, uint64_t b, uint64_t prime, int32_t n_hash,
                                 int32_t rows_per_band, unsigned long long* keys,
                                 void* out, int32_t out_dtype, int32_t write_signatures, int32_t* status,
                                 void* workspace, size_t workspace_bytes, void* stream);

/*
 * Random family with 64-bit parameters (a, b: device uint64[n_hash]), required for
 * primes >= 2^31; any prime < 2^63.  No workspace.
 */
int mhb_sign_random_csr_u64(const int64_t* indptr, const uint32_t* ids,
                            int64_t n_sets, int64_t nnz,
                            const uint64_t* a, const uint64_t* b, uint64_t prime, int32_t n_hash,
                            void* out, int32_t out_dtype, int32_t* status, void* stream);

/*
 * 64-bit feature ids (the reference's FeatureSet ids are int64: with a prime >= 2^32
 * they may reach p - 1, minhash.py:99-127).  kind 0 iterative (a, b), 1 random
 * (ra, rb: device uint64[n_hash]); any prime < 2^63; ids: device uint64[nnz];
 * out: device int64[n_sets * n_hash].  Runs the 64-bit-residue path (wide.cu).
 */
int mhb_sign_csr_ids64(int32_t kind, const int64_t* indptr, const uint64_t* ids, int64_t n_sets, int64_t nnz,
                       uint64_t a, uint64_t b, const uint64_t* ra, const uint64_t* rb, uint64_t prime,
                       int32_t n_hash, long long* out, int32_t* status, void* stream);

/*
 * Host-buffer entry (the end-to-end path an FFI caller uses): indptr/ids/out are
 * HOST pointers (page-locked for full copy bandwidth; pageable also works).  The
 * library stages chunks through its own device buffers on `device` with copy/
 * compute overlap, and returns when out is complete.  kind: 0 iterative, 1 random
 * (a_host/b_host used for random, a/b scalars for iterative; a_host/b_host may also be
 * device arrays -- UVA tells them apart -- and are then used in place).  device -1: the
 * calling thread's current CUDA device.
 * Small batches (<= 64 sets, the per-set reference call) take no launch: a resident
 * block polling mapped host memory serves them (the "doorbell"; it exits after
 * MHB_DOORBELL_IDLE_US, default 1000, of no requests; MHB_DOORBELL=0 launches a
 * kernel per call instead).
 */
int mhb_sign_csr_host(int32_t kind, const int64_t* indptr, const uint32_t* ids,
                      int64_t n_sets, int64_t nnz,
                      uint64_t a, uint64_t b, const uint32_t* a_host, const uint32_t* b_host,
                      uint64_t prime, int32_t n_hash,
                      void* out, int32_t out_dtype, int32_t* status_host, int32_t device);

/* Release the device buffers and streams cached by mhb_sign_csr_host. */
void mhb_host_release(void);

/*
 * Diagnostic (no GPU needed): runs `jobs` back-to-back jobs of 2..64 parts on the host
 * copy pool mhb_sign_csr_host stages pageable buffers with, from `threads` concurrent
 * callers, each part recording how often it ran.  *bad = parts that ran other than
 * exactly once (0 for a correct pool).  Returns MHB_OK.
 */
int mhb_host_pool_selftest(int64_t jobs, uint64_t seed, int32_t threads, int64_t* bad);

/*
 * Pairwise Jaccard estimates for listed pairs (replaces estimate_jaccard,
 * minhash.py:130-137): counts[k] = #{i : sig[pi[k]][i] == sig[pj[k]][i]};
 * est[k] = (double)counts[k] / n_hash (IEEE division, bit-identical to numpy's
 * mean of the 0/1 vector for n_hash < 2^53).  est may be NULL.
 */
int mhb_jaccard_pairs(const void* sig, int32_t sig_dtype, int32_t n_hash,
                      const int64_t* pi, const int64_t* pj, int64_t n_pairs,
                      uint32_t* counts, double* est, void* stream);

/*
 * Block x block estimates: counts[r*n_cols + c] = #{i : A[r][i] == B[c][i]} for
 * signature blocks A (n_rows x n_hash) and B (n_cols x n_hash) of dtype sig_dtype.
 */
int mhb_jaccard_block(const void* sig_a, int64_t n_rows, const void* sig_b, int64_t n_cols,
                      int32_t sig_dtype, int32_t n_hash, uint32_t* counts, void* stream);

/*
 * LSH band keys (the reference has no banding): the N
 * signature positions form N/rows_per_band bands of consecutive rows, and
 *   keys[s*n_bands + band] = splitmix64(h1 << 32 | h2), where over the band's argmin ids x
 *   (uint32, row order) h1 <- h1*0x9E3779B1 + x and h2 <- h2*0x85EBCA6B + x (mod 2^32),
 *   seeded h1 = 0x811C9DC5 ^ band, h2 = 0xC2B2AE35 ^ (band*0x27D4EB2F) (csrc/bandhash.cuh:
 *   two IMADs per id, so the signing epilogue hashes its bands off the ALU pipe).
 * sig: [n_sets, n_hash] of sig_dtype; rows_per_band must divide n_hash.
 */
int mhb_band_keys(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                  int32_t rows_per_band, unsigned long long* keys, void* stream);

/*
 * Bucket-uniformity histogram (generalises stats.py:221-224 from one x to a
 * batch): counts[m] += #{(x, i) : x in xs, 0 <= i < n_hash, h_i(x) mod buckets == m}.
 * counts is uint64[buckets], accumulated into (not cleared).  xs must be < prime.
 */
int mhb_bucket_hist_iterative(const uint32_t* xs, int64_t n_x,
                              uint64_t a, uint64_t b, uint64_t prime, int32_t n_hash,
                              uint32_t buckets, unsigned long long* counts, void* stream);
int mhb_bucket_hist_random(const uint32_t* xs, int64_t n_x,
                           const uint32_t* a, const uint32_t* b, uint64_t prime, int32_t n_hash,
                           uint32_t buckets, unsigned long long* counts, void* stream);
/*
 * The same counts for any prime up to 2^63 (families.py:105-112 counts for every
 * prime): kind 0 = iterative (a, b), kind 1 = random (device uint64 arrays ra, rb);
 * xs are uint64 (< prime).  64-bit residues; the u32 entries above route iterative
 * families with 2^31 <= prime here themselves.
 */
int mhb_bucket_hist_u64(int32_t kind, const uint64_t* xs, int64_t n_x, uint64_t a, uint64_t b,
                        const uint64_t* ra, const uint64_t* rb, uint64_t prime, int32_t n_hash,
                        uint64_t buckets, unsigned long long* counts, void* stream);

/*
 * Signature-file records from a device signature block (the reference's formats,
 * minhash.py:140-206).  obj_ids (device int64[n_sets]) may be NULL: ids are then
 * first_id, first_id+1, ...
 *   binary: out is uint64[n_sets*(n_hash+2)]: per record id, n_hash, then the ids
 *           (little-endian, byte-identical to write_signatures_binary).
 *   text  : lens[r] = byte length of record r's line "id N x0 ... xN-1\n"; after an
 *           exclusive scan of lens into offsets, format_text writes the lines into
 *           out (byte-identical to write_signatures_text).
 */
int mhb_format_binary_records(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                              const int64_t* obj_ids, int64_t first_id, unsigned long long* out, void* stream);
int mhb_text_record_lengths(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                            const int64_t* obj_ids, int64_t first_id, int64_t* lens, void* stream);
int mhb_format_text_records(const void* sig, int32_t sig_dtype, int64_t n_sets, int32_t n_hash,
                            const int64_t* obj_ids, int64_t first_id, const int64_t* offsets, char* out,
                            void* stream);

/*
 * Corpus ingest (reference corpus.py:18-80: build_corpus, tokenize, Vocabulary):
 * a one-document-per-line UTF-8 buffer -> CSR feature ids + vocabulary.
 *   lines   : "\n", "\r\n" or a lone "\r" end a line (Python universal newlines);
 *   terms   : lowercase maximal alphanumeric runs ([^\W_]), deduplicated, sorted;
 *   ids     : vocabulary ids in first-occurrence order (document order, then the
 *             document's sorted terms); each document is its sorted id set.
 * Host backend multi-threaded (n_threads <= 0: all hardware threads); device backend:
 * mhb_corpus_scan_device.  Lines with a byte >= 0x80 are "deferred": their pure-ASCII
 * segments (maximal runs of [A-Za-z0-9\x80-\xff] without a byte >= 0x80) are tokenized
 * natively, and the caller supplies, through mhb_corpus_set_terms before
 * mhb_corpus_intern, the terms of the line's other segments -- tokenize() of those
 * segments joined by "\n", with Python's Unicode str.lower / str.isalnum -- or of the
 * whole line when it holds U+03A3 (bytes CE A3; Final_Sigma is the one lowercase rule
 * that looks across separators).  `text` must stay alive and unchanged until
 * mhb_corpus_free.
 */
typedef struct mhb_corpus mhb_corpus;
int mhb_corpus_scan(const char* text, int64_t n_bytes, int32_t n_threads, mhb_corpus** corpus);
/* Unicode tables of the caller's Python (what tokenize() uses): bit c of alnum_bits is
   chr(c).isalnum(); lower_keys (ascending) are the code points whose str.lower() differs,
   lower_vals[3k..3k+2] the lowercase code points of lower_keys[k] (0xFFFFFFFF padded);
   cased_bits / ignorable_bits (optional) are the Cased and Case_Ignorable properties that
   str.lower() consults for U+03A3 (Final_Sigma). */
typedef struct mhb_unicode_tables {
    const uint32_t* alnum_bits;      /* [0x110000 / 32] */
    const uint32_t* lower_keys;      /* [n_lower] */
    const uint32_t* lower_vals;      /* [3 * n_lower] */
    int32_t n_lower;
    const uint32_t* cased_bits;      /* [0x110000 / 32] or NULL */
    const uint32_t* ignorable_bits;  /* [0x110000 / 32] or NULL */
} mhb_unicode_tables;
/* The same ingest on GPU `device` (corpus_gpu.cu): lines, tokens, vocabulary and documents are
   computed on the device; the rest of the mhb_corpus_* API is shared.  `text` is a host buffer
   (pinned for full PCIe speed).  With `tables`, lines holding non-ASCII bytes are tokenized on the
   device too (strict UTF-8, full lowercase mapping incl. Final_Sigma, isalnum), except lines with
   invalid UTF-8 (and, without cased/ignorable bits, lines with U+03A3), which stay deferred to the
   caller under the rule above; tables == NULL defers every non-ASCII segment as the host backend
   does. */
int mhb_corpus_scan_device(const char* text, int64_t n_bytes, int32_t device, const mhb_unicode_tables* tables,
                           mhb_corpus** corpus);
int mhb_corpus_info(const mhb_corpus* corpus, int64_t* n_docs, int64_t* n_deferred);
/* per deferred line k: its document index, byte offset and byte length in `text` */
int mhb_corpus_deferred(const mhb_corpus* corpus, int64_t* lines, int64_t* starts, int64_t* lens);
/* terms of deferred line lines[k] are term_offsets[line_ptr[k] .. line_ptr[k+1]] slices of blob */
int mhb_corpus_set_terms(mhb_corpus* corpus, int64_t n_lines, const int64_t* lines, const int64_t* line_ptr,
                         const char* blob, const int64_t* term_offsets);
int mhb_corpus_intern(mhb_corpus* corpus, int64_t* nnz, int64_t* n_terms, int64_t* term_bytes,
                      int64_t* empty_docs);
/* indptr int64[n_docs+1], ids uint32[nnz]; the vocabulary in id order as term_blob char[term_bytes]
   (each term followed by '\n') with term_offsets int64[n_terms+1] (term starts, then term_bytes);
   any pointer may be NULL */
int mhb_corpus_export(const mhb_corpus* corpus, int64_t* indptr, uint32_t* ids, int64_t* term_offsets,
                      char* term_blob);
/* device-backend handles: copy indptr / ids into device buffers on `stream` (feeds mhb_sign_*_csr) */
int mhb_corpus_export_device(const mhb_corpus* corpus, int64_t* indptr, uint32_t* ids, void* stream);
void mhb_corpus_free(mhb_corpus* corpus);

/*
 * Peer-memory gather target (fused sign + gather across ranks, one process per GPU).
 * mhb_peer_alloc: cudaMalloc `bytes` on `device` and export its 64-byte CUDA IPC handle.
 * mhb_peer_open: map another process's buffer (NVLink peer mapping across GPUs); any
 * mhb_sign_* entry may then take out = mapped + row0 * n_hash * elem_size and its
 * stores land directly in the owner's matrix.  Close / free when every writer's
 * stream has completed (a barrier after the sign calls).
 */
int mhb_peer_alloc(size_t bytes, int32_t device, void** ptr, unsigned char handle[64]);
int mhb_peer_open(const unsigned char handle[64], int32_t device, void** ptr);
int mhb_peer_close(void* ptr);
int mhb_peer_free(void* ptr);

/*
 * Instruction-rate probe for the roofline: runs a visit sequence from registers only,
 * `visits_per_thread` visits per thread on a persistent grid, and reports visits and
 * device ms.  kind 0: iterative (add, conditional subtract, 3-way min); 1: random family,
 * Shoup lanes; 2: random family, float-quotient lanes (the kernel's path for p <= 2^23).
 */
int mhb_probe_visit_rate(int64_t visits_per_thread, int32_t kind,
                         double* visits_out, float* ms_out, void* stream);

/*
 * Kernel timing for benchmarks: while enabled, every mhb_sign_* call records a CUDA
 * event pair on its stream around the main signature kernel (up to max_launches
 * calls).  mhb_profile_end synchronises on the recorded events and returns the
 * summed device time of the main kernel and the number of launches timed.
 */
int mhb_profile_begin(int32_t max_launches);
int mhb_profile_end(float* total_ms, int32_t* n_launches);

#ifdef __cplusplus
}
#endif

#endif /* MHB_H_ */
