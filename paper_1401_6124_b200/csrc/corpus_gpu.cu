// corpus_gpu.cu -- corpus ingest on the GPU (device backend of mhb_corpus_*).
//
// Same result as corpus.cpp and as the reference's build_corpus (src/corpus.py:67-80):
// universal-newline lines, lowercase alphanumeric runs deduplicated per line,
// vocabulary ids in first-occurrence order, documents as sorted id sets.  With the
// caller's Unicode tables (mhb_unicode_tables: this Python's str.isalnum / str.lower and
// the Cased / Case_Ignorable sets of its Final_Sigma rule), lines holding non-ASCII
// bytes are tokenized here as well (uni_lines); only lines with invalid UTF-8 are
// deferred, and without tables the non-ASCII segments are deferred as in the host
// backend.  Deferred terms come back through mhb_corpus_set_terms and are spliced in
// at their line, so every later step sees the tokens in document order.
//
// Pipeline (one private stream, CUB device primitives + the kernels below):
//   scan    break positions (universal newlines) -> line [start, end); one warp per
//           line counts token starts and flags non-ASCII lines.
//   intern  tokens in document order (warp per line; deferred lines copy their
//           supplied terms) -> 64-bit hash of the lowercased bytes -> stable radix
//           sort by hash.  Equal hashes form runs; every token is compared byte for
//           byte with its predecessor in the run (a collision re-hashes with a new
//           seed), so the grouping is exact.  Stability makes a run's head its
//           earliest token, hence the term's first line.  Vocabulary order is
//           (first line, term bytes): two stable radix sorts on (8-byte big-endian
//           prefix, first line) and an insertion-sort fix-up of the rare groups that
//           tie on both.  Documents: per-line segmented sort of the ids, unique, CSR.
// Every byte and index is exact; no floating point.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "common.h"
#include "corpus_device.h"

namespace mhb {

namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ bool is_alnum(uint8_t c) {
    return (uint8_t)((c | 0x20) - 'a') < 26 || (uint8_t)(c - '0') < 10;
}
__device__ __forceinline__ uint8_t to_lower(uint8_t c) { return (uint8_t)(c - 'A') < 26 ? c + 32 : c; }

struct Src {  // token bytes live in the text or, for deferred lines, in the supplied blob
    const uint8_t* text;
    const uint8_t* blob;
    int64_t n_bytes;
    __device__ __forceinline__ const uint8_t* at(int64_t start) const {
        return start < n_bytes ? text + start : blob + (start - n_bytes);
    }
};

struct IsBreak {
    const uint8_t* s;
    __device__ __forceinline__ bool operator()(int64_t j) const {
        const uint8_t c = s[j];
        return c == '\r' || (c == '\n' && !(j > 0 && s[j - 1] == '\r'));
    }
};

struct BreakFlag {
    const uint8_t* s;
    __device__ __forceinline__ int64_t operator()(int64_t j) const { return IsBreak{s}(j) ? 1 : 0; }
};

__global__ void lines_from_breaks(const int64_t* brk, int64_t n_brk, const uint8_t* s, int64_t n,
                                  int64_t* line_start, int64_t* line_end) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k == 0) line_start[0] = 0;
    if (k < n_brk) {
        const int64_t j = brk[k];
        line_end[k] = j;
        line_start[k + 1] = j + ((s[j] == '\r' && j + 1 < n && s[j + 1] == '\n') ? 2 : 1);
    }
    if (k == n_brk) line_end[n_brk] = n;  // used only when the last line has no terminator
}

// A native token is a maximal ASCII alphanumeric run whose neighbours are not
// non-ASCII bytes (its segment -- maximal run of [A-Za-z0-9\x80-\xff] -- is pure
// ASCII).  Lines holding U+03A3 (bytes CE A3: Python's only context-dependent
// lowercase, Final_Sigma) have no native tokens; their caller supplies every term.
__device__ __forceinline__ bool native_start(const uint8_t* s, int64_t j, int64_t s1, int64_t* end) {
    if (j >= s1 || !is_alnum(s[j])) return false;
    if (j > 0 && (is_alnum(s[j - 1]) || s[j - 1] >= 0x80)) return false;
    int64_t e = j + 1;
    while (e < s1 && is_alnum(s[e])) ++e;
    *end = e;
    return !(e < s1 && s[e] >= 0x80);
}

// One warp per line: native token count, non-ASCII and U+03A3 detection.
__global__ void scan_lines(const uint8_t* s, const int64_t* line_start, const int64_t* line_end, int64_t n_docs,
                           int64_t* ncount, uint8_t* deferred, bool uni) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t d = w0; d < n_docs; d += nw) {
        const int64_t s0 = line_start[d], s1 = line_end[d];
        int64_t cnt = 0;
        bool foreign = false, sigma = false;
        for (int64_t b = s0; b < s1; b += 32) {
            const int64_t j = b + lane;
            const uint8_t c = j < s1 ? s[j] : (uint8_t)' ';
            foreign |= __any_sync(0xffffffffu, c >= 0x80);
            sigma |= __any_sync(0xffffffffu, c == 0xCE && j + 1 < s1 && s[j + 1] == 0xA3);
            int64_t e;
            cnt += __popc(__ballot_sync(0xffffffffu, native_start(s, j, s1, &e)));
        }
        if (lane == 0) {
            deferred[d] = foreign ? 1 : 0;
            ncount[d] = (sigma || (uni && foreign)) ? 0 : cnt;  // uni: uni_lines tokenizes the whole line
        }
    }
}

__global__ void scatter_deferred(const int64_t* lines, const int64_t* cnt, const int64_t* first, int64_t n,
                                 int64_t* scount, int64_t* dfirst) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) {
        scount[lines[k]] = cnt[k];
        dfirst[lines[k]] = first[k];
    }
}

__global__ void add_counts(const int64_t* a, const int64_t* b, const int64_t* c, int64_t n, int64_t* out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = a[k] + b[k] + c[k];
}

// One warp per line: token (start, len, line) in document order -- the line's native
// tokens, then (deferred lines) the caller-supplied terms.
__global__ void write_tokens(const uint8_t* s, int64_t n_bytes, const int64_t* line_start, const int64_t* line_end,
                             int64_t n_docs, const int64_t* ncount, const uint8_t* code, const int64_t* tok_off,
                             const int64_t* dfirst, const int64_t* dterm_off, int64_t* tok_start, uint32_t* tok_len,
                             uint32_t* tok_line) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t d = w0; d < n_docs; d += nw) {
        const int64_t t0 = tok_off[d], nn = ncount[d];
        if (nn) {
            const int64_t s0 = line_start[d], s1 = line_end[d];
            int64_t rank = 0;
            for (int64_t b = s0; b < s1; b += 32) {
                const int64_t j = b + lane;
                int64_t e = 0;
                const bool st = native_start(s, j, s1, &e);
                const unsigned m = __ballot_sync(0xffffffffu, st);
                if (st) {
                    const int64_t t = t0 + rank + __popc(m & ((1u << lane) - 1));
                    tok_start[t] = j;
                    tok_len[t] = (uint32_t)(e - j);
                    tok_line[t] = (uint32_t)d;
                }
                rank += __popc(m);
            }
        }
        const int64_t ns = code[d] == 1 ? tok_off[d + 1] - t0 - nn : 0;  // caller-supplied terms
        if (ns > 0) {
            const int64_t k0 = dfirst[d];
            for (int64_t r = lane; r < ns; r += 32) {
                tok_start[t0 + nn + r] = n_bytes + dterm_off[k0 + r];
                tok_len[t0 + nn + r] = (uint32_t)(dterm_off[k0 + r + 1] - dterm_off[k0 + r]);
                tok_line[t0 + nn + r] = (uint32_t)d;
            }
        }
    }
}

// 64-bit hash of the lowercased bytes (seeded) and the 8-byte big-endian prefix.
__global__ void hash_tokens(Src src, const int64_t* tok_start, const uint32_t* tok_len, int64_t n_tok, uint64_t seed,
                            unsigned long long* h_out, unsigned long long* key_out, uint32_t* idx_out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_tok) return;
    const uint8_t* p = src.at(tok_start[t]);
    const uint32_t n = tok_len[t];
    uint64_t h = seed ^ 0x9E3779B97F4A7C15ull ^ ((uint64_t)n * 0xFF51AFD7ED558CCDull);
    uint64_t w = 0, key = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const uint64_t c = to_lower(p[i]);
        w |= c << (8 * (i & 7));
        if (i < 8) key |= c << (8 * (7 - i));
        if ((i & 7) == 7) {
            h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
            h ^= h >> 29;
            w = 0;
        }
    }
    h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 32;
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 29;
    h_out[t] = h;
    key_out[t] = key;
    idx_out[t] = (uint32_t)t;
}

__device__ __forceinline__ bool same_term(const Src& src, int64_t sa, uint32_t la, int64_t sb, uint32_t lb) {
    if (la != lb) return false;
    const uint8_t* a = src.at(sa);
    const uint8_t* b = src.at(sb);
    for (uint32_t i = 0; i < la; ++i)
        if (to_lower(a[i]) != to_lower(b[i])) return false;
    return true;
}

// Run heads over the hash-sorted tokens; every non-head is verified against its predecessor.
__global__ void run_heads(Src src, const unsigned long long* hs, const uint32_t* order, const int64_t* tok_start,
                          const uint32_t* tok_len, int64_t n_tok, uint32_t* head, int* collision) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_tok) return;
    const bool h = i == 0 || hs[i] != hs[i - 1];
    head[i] = h ? 1u : 0u;
    if (!h) {
        const uint32_t a = order[i], b = order[i - 1];
        if (!same_term(src, tok_start[a], tok_len[a], tok_start[b], tok_len[b])) atomicOr(collision, 1);
    }
}

__global__ void run_info(const uint32_t* head, const uint32_t* run_incl, const uint32_t* order,
                         const uint32_t* tok_line, const unsigned long long* tok_key, int64_t n_tok,
                         uint32_t* run_of_tok, uint32_t* run_tok, uint32_t* run_line, unsigned long long* run_key,
                         uint32_t* run_idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_tok) return;
    const uint32_t r = run_incl[i] - 1;
    const uint32_t t = order[i];
    run_of_tok[t] = r;
    if (head[i]) {  // stable sort: the head is the run's earliest token -> its first line
        run_tok[r] = t;
        run_line[r] = tok_line[t];
        run_key[r] = tok_key[t];
        run_idx[r] = r;
    }
}

__global__ void gather_u32(const uint32_t* src, const uint32_t* idx, int64_t n, uint32_t* dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

__device__ __forceinline__ bool term_less(const Src& src, int64_t sa, uint32_t la, int64_t sb, uint32_t lb) {
    const uint8_t* a = src.at(sa);
    const uint8_t* b = src.at(sb);
    const uint32_t n = la < lb ? la : lb;
    for (uint32_t i = 0; i < n; ++i) {
        const uint8_t x = to_lower(a[i]), y = to_lower(b[i]);
        if (x != y) return x < y;
    }
    return la < lb;
}

// Groups of runs tying on (first line, 8-byte prefix) are put in full byte order.
__global__ void fix_ties(Src src, uint32_t* order, const uint32_t* run_line, const unsigned long long* run_key,
                         const uint32_t* run_tok, const int64_t* tok_start, const uint32_t* tok_len, int64_t U) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= U) return;
    auto tie = [&](int64_t i) {
        return i > 0 && i < U && run_line[order[i]] == run_line[order[i - 1]] && run_key[order[i]] == run_key[order[i - 1]];
    };
    if (tie(g) || !tie(g + 1)) return;  // g starts a tie group
    int64_t e = g + 1;
    while (tie(e)) ++e;
    for (int64_t i = g + 1; i < e; ++i) {  // insertion sort by full bytes
        const uint32_t v = order[i];
        const int64_t sv = tok_start[run_tok[v]];
        const uint32_t lv = tok_len[run_tok[v]];
        int64_t j = i;
        while (j > g) {
            const uint32_t u = order[j - 1];
            if (!term_less(src, sv, lv, tok_start[run_tok[u]], tok_len[run_tok[u]])) break;
            order[j] = u;
            --j;
        }
        order[j] = v;
    }
}

__global__ void assign_ids(const uint32_t* order, const uint32_t* run_tok, const uint32_t* tok_len, int64_t U,
                           uint32_t* id_of_run, int64_t* term_len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < U) {
        id_of_run[order[i]] = (uint32_t)i;
        term_len[i] = (int64_t)tok_len[run_tok[order[i]]] + 1;  // + '\n'
    }
    if (i == U) term_len[U] = 0;
}

__global__ void write_vocab(Src src, const uint32_t* order, const uint32_t* run_tok, const int64_t* tok_start,
                            const uint32_t* tok_len, const int64_t* voff, int64_t U, char* blob) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= U) return;
    const uint32_t t = run_tok[order[i]];
    const uint8_t* p = src.at(tok_start[t]);
    char* o = blob + voff[i];
    const uint32_t n = tok_len[t];
    for (uint32_t k = 0; k < n; ++k) o[k] = (char)to_lower(p[k]);
    o[n] = '\n';
}

__global__ void token_ids(const uint32_t* run_of_tok, const uint32_t* id_of_run, int64_t n_tok, uint32_t* ids) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n_tok) ids[t] = id_of_run[run_of_tok[t]];
}

__global__ void unique_flags(const uint32_t* sorted, const uint32_t* tok_line, const int64_t* tok_off, int64_t n_tok,
                             int64_t* keep) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n_tok) keep[i] = (i == tok_off[tok_line[i]] || sorted[i] != sorted[i - 1]) ? 1 : 0;
    if (i == n_tok) keep[n_tok] = 0;
}

__global__ void compact_csr(const uint32_t* sorted, const int64_t* keep, const int64_t* pos, const int64_t* tok_off,
                            int64_t n_tok, int64_t n_docs, uint32_t* ids_out, int64_t* indptr,
                            unsigned long long* empty) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n_tok && keep[i]) ids_out[pos[i]] = sorted[i];
    if (i <= n_docs) {
        indptr[i] = pos[tok_off[i]];
        if (i < n_docs && tok_off[i + 1] == tok_off[i]) atomicAdd(empty, 1ull);
    }
}

// ---- Unicode lines on the device ---------------------------------------------------
// With the caller's tables (str.isalnum / str.lower of the running Python), a line
// holding non-ASCII bytes is tokenized here exactly as tokenize() does it: strict
// UTF-8 decode, lowercase each code point (full mapping, 1..3 code points), tokens =
// maximal runs of alphanumeric lowered code points, re-encoded as UTF-8.  Lines with
// invalid UTF-8 (the reference raises) or U+03A3 (Final_Sigma, context-dependent)
// stay deferred to the caller.
struct UniTab {
    const uint32_t* alnum;  // bitmap over code points
    const uint32_t* keys;   // ascending code points whose lowercase differs
    const uint32_t* vals;   // [n * 3] lowercase code points, 0xFFFFFFFF padded
    int n;
    const uint32_t* cased;      // Final_Sigma context (nullptr: U+03A3 lines stay deferred)
    const uint32_t* ignorable;
};

__device__ __forceinline__ bool uni_bit(const uint32_t* b, uint32_t c) { return (b[c >> 5] >> (c & 31)) & 1u; }

__device__ __forceinline__ bool uni_alnum(const UniTab& t, uint32_t c) { return (t.alnum[c >> 5] >> (c & 31)) & 1u; }

__device__ __forceinline__ int uni_lower(const UniTab& t, uint32_t cp, uint32_t* out) {
    if (cp < 0x80) {
        out[0] = (cp - 'A' < 26u) ? cp + 32 : cp;
        return 1;
    }
    int lo = 0, hi = t.n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (t.keys[mid] < cp) lo = mid + 1;
        else hi = mid;
    }
    if (lo < t.n && t.keys[lo] == cp) {
        int k = 0;
        for (; k < 3 && t.vals[3 * lo + k] != 0xFFFFFFFFu; ++k) out[k] = t.vals[3 * lo + k];
        return k;
    }
    out[0] = cp;
    return 1;
}

// Strict UTF-8 (Python's decoder): no overlongs, surrogates or code points > U+10FFFF.
__device__ __forceinline__ int utf8_decode(const uint8_t* s, int64_t i, int64_t end, uint32_t* cp) {
    const uint32_t b0 = s[i];
    if (b0 < 0x80) {
        *cp = b0;
        return 1;
    }
    int n;
    uint32_t lo = 0x80, hi = 0xBF, c;
    if (b0 >= 0xC2 && b0 <= 0xDF) {
        n = 2;
        c = b0 & 0x1F;
    } else if (b0 >= 0xE0 && b0 <= 0xEF) {
        n = 3;
        c = b0 & 0x0F;
        if (b0 == 0xE0) lo = 0xA0;
        if (b0 == 0xED) hi = 0x9F;
    } else if (b0 >= 0xF0 && b0 <= 0xF4) {
        n = 4;
        c = b0 & 0x07;
        if (b0 == 0xF0) lo = 0x90;
        if (b0 == 0xF4) hi = 0x8F;
    } else {
        return 0;
    }
    if (i + n > end) return 0;
    for (int k = 1; k < n; ++k) {
        const uint32_t b = s[i + k];
        if (k == 1 ? (b < lo || b > hi) : (b < 0x80 || b > 0xBF)) return 0;
        c = (c << 6) | (b & 0x3F);
    }
    *cp = c;
    return n;
}

// Python's handle_capital_sigma (Objects/unicodeobject.c): U+03A3 lowercases to U+03C2
// when a cased letter precedes it and none follows, skipping case-ignorable code points,
// within the string being lowered -- here the line.  `at` is the byte offset of the
// U+03A3; earlier code points of the line are already validated.  Returns 0 on invalid
// UTF-8 after it.
__device__ __forceinline__ uint32_t final_sigma(const UniTab& t, const uint8_t* s, int64_t s0, int64_t s1, int64_t at) {
    bool fin = false;
    for (int64_t j = at; j > s0;) {  // backward
        int64_t k = j - 1;
        while (k > s0 && (s[k] & 0xC0) == 0x80) --k;
        uint32_t c;
        utf8_decode(s, k, s1, &c);
        if (!uni_bit(t.ignorable, c)) {
            fin = uni_bit(t.cased, c);
            break;
        }
        j = k;
    }
    if (fin) {  // forward
        for (int64_t k = at + 2; k < s1;) {
            uint32_t c;
            const int len = utf8_decode(s, k, s1, &c);
            if (!len) return 0;
            if (!uni_bit(t.ignorable, c)) {
                fin = !uni_bit(t.cased, c);
                break;
            }
            k += len;
        }
    }
    return fin ? 0x3C2u : 0x3C3u;
}

__device__ __forceinline__ int utf8_len(uint32_t c) { return c < 0x80 ? 1 : c < 0x800 ? 2 : c < 0x10000 ? 3 : 4; }

__device__ __forceinline__ void utf8_put(uint8_t* o, uint32_t c) {
    if (c < 0x80) {
        o[0] = (uint8_t)c;
    } else if (c < 0x800) {
        o[0] = (uint8_t)(0xC0 | (c >> 6));
        o[1] = (uint8_t)(0x80 | (c & 0x3F));
    } else if (c < 0x10000) {
        o[0] = (uint8_t)(0xE0 | (c >> 12));
        o[1] = (uint8_t)(0x80 | ((c >> 6) & 0x3F));
        o[2] = (uint8_t)(0x80 | (c & 0x3F));
    } else {
        o[0] = (uint8_t)(0xF0 | (c >> 18));
        o[1] = (uint8_t)(0x80 | ((c >> 12) & 0x3F));
        o[2] = (uint8_t)(0x80 | ((c >> 6) & 0x3F));
        o[3] = (uint8_t)(0x80 | (c & 0x3F));
    }
}

// Thread per non-ASCII line.  COUNT: tokens and lowered token bytes, or "stay deferred"
// (code 1) for invalid UTF-8 (or U+03A3 without the Final_Sigma tables); handled lines
// become code 3.  WRITE: the tokens
// (start into the blob region, length, line) and their lowered bytes.
template <bool WRITE>
__global__ void uni_lines(const uint8_t* s, const int64_t* line_start, const int64_t* line_end, int64_t n_docs,
                          UniTab tab, uint8_t* code, int64_t* ucount, int64_t* ubytes, const int64_t* tok_off,
                          const int64_t* uoff, int64_t blob_base, uint8_t* ubuf, int64_t* tok_start,
                          uint32_t* tok_len, uint32_t* tok_line) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n_docs;
         d += (int64_t)gridDim.x * blockDim.x) {
        if (code[d] != (WRITE ? 3 : 1)) continue;
        const int64_t s0 = line_start[d], s1 = line_end[d];
        int64_t cnt = 0, nb = 0, tok0 = 0;
        bool in_tok = false, bad = false;
        const int64_t t0 = WRITE ? tok_off[d] : 0;
        uint8_t* o = WRITE ? ubuf + uoff[d] : nullptr;
        for (int64_t i = s0; i < s1;) {
            uint32_t cp;
            const int len = utf8_decode(s, i, s1, &cp);
            if (!len || (cp == 0x3A3 && !tab.cased)) {
                bad = true;
                break;
            }
            uint32_t lc[3];
            int m;
            if (cp == 0x3A3) {
                lc[0] = final_sigma(tab, s, s0, s1, i);
                m = 1;
                if (!lc[0]) {
                    bad = true;
                    break;
                }
            } else {
                m = uni_lower(tab, cp, lc);
            }
            i += len;
            for (int k = 0; k < m; ++k) {
                if (uni_alnum(tab, lc[k])) {
                    if (!in_tok) {
                        in_tok = true;
                        tok0 = nb;
                    }
                    if (WRITE) utf8_put(o + nb, lc[k]);
                    nb += utf8_len(lc[k]);
                } else if (in_tok) {
                    in_tok = false;
                    if (WRITE) {
                        tok_start[t0 + cnt] = blob_base + uoff[d] + tok0;
                        tok_len[t0 + cnt] = (uint32_t)(nb - tok0);
                        tok_line[t0 + cnt] = (uint32_t)d;
                    }
                    ++cnt;
                }
            }
        }
        if (!WRITE && bad) continue;  // stays deferred (code 1)
        if (in_tok) {
            if (WRITE) {
                tok_start[t0 + cnt] = blob_base + uoff[d] + tok0;
                tok_len[t0 + cnt] = (uint32_t)(nb - tok0);
                tok_line[t0 + cnt] = (uint32_t)d;
            }
            ++cnt;
        }
        if (!WRITE) {
            code[d] = 3;
            ucount[d] = cnt;
            ubytes[d] = nb;
        }
    }
}

inline unsigned blocks_for(int64_t n, int threads = 256) { return (unsigned)((n + threads - 1) / threads + 1); }
inline unsigned warp_blocks(int64_t n_docs) {
    const int64_t b = (n_docs + kWarpsPerBlock - 1) / kWarpsPerBlock;
    return (unsigned)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 64);
}

// Device scratch owned by one call; freed stream-ordered.
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    template <typename T>
    T* get(size_t n) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st) != cudaSuccess) throw std::bad_alloc();
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

// MHB_CORPUS_TIMING=1: per-stage wall times (stream-synchronised) on stderr.
struct StageTimer {
    cudaStream_t st;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit StageTimer(cudaStream_t s) : st(s), on(false) {
        const char* e = std::getenv("MHB_CORPUS_TIMING");
        on = e && e[0] && e[0] != '0';
        t = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[corpus_gpu] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

#define MHB_CUDA(x)                                          \
    do {                                                     \
        cudaError_t e_ = (x);                                \
        if (e_ != cudaSuccess) return cuda_check(e_, #x);    \
    } while (0)

}  // namespace

struct CorpusDevice {
    int device = 0;
    cudaStream_t st = nullptr;
    int64_t n_bytes = 0, n_docs = 0;
    uint8_t* text = nullptr;       // device copy of the text
    int64_t* line_start = nullptr;  // [n_docs + 1]
    int64_t* line_end = nullptr;
    int64_t* count = nullptr;       // [n_docs + 1] native tokens per line
    uint8_t* deferred = nullptr;    // [n_docs] 0 ASCII, 1 deferred to the caller, 3 Unicode on the device
    std::vector<uint8_t> deferred_h;
    // Unicode tables (device copies) and per-line Unicode token counts / lowered bytes
    bool uni = false;
    UniTab tab{};
    uint32_t* tab_buf = nullptr;
    int64_t* ucount = nullptr;      // [n_docs + 1]
    int64_t* ubytes = nullptr;      // [n_docs + 1]
    // supplied terms of the deferred lines (host until intern)
    std::vector<int64_t> dl_line, dl_cnt, dl_first, dterm_off{0};
    std::vector<char> dblob;
    // results
    bool interned = false;
    int64_t nnz = 0, n_terms = 0, term_bytes = 0, empty = 0;
    int64_t* indptr = nullptr;
    uint32_t* ids = nullptr;
    int64_t* voff = nullptr;
    char* vblob = nullptr;
    // device buffers are stream-ordered allocations on `st` (no device-wide sync on free)
    template <typename T>
    cudaError_t alloc(T** p, size_t n) {
        return cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), st);
    }
    ~CorpusDevice() {
        if (!st) return;
        cudaSetDevice(device);
        for (void* p : {(void*)text, (void*)line_start, (void*)line_end, (void*)count, (void*)deferred,
                        (void*)indptr, (void*)ids, (void*)voff, (void*)vblob, (void*)tab_buf, (void*)ucount,
                        (void*)ubytes})
            if (p) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
};

int corpus_device_scan(const char* text_h, int64_t n, int device, const mhb_unicode_tables* tables,
                       CorpusDevice** out, std::vector<int64_t>& line_start, std::vector<int64_t>& line_end,
                       std::vector<int64_t>& deferred_lines) {
    MHB_CUDA(cudaSetDevice(device));
    auto d = std::make_unique<CorpusDevice>();
    d->device = device;
    d->n_bytes = n;
    MHB_CUDA(cudaStreamCreateWithFlags(&d->st, cudaStreamNonBlocking));
    cudaStream_t st = d->st;
    {  // keep the stream-ordered pool's memory mapped between calls (no re-faulting per ingest)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    StageTimer tm(st);
    MHB_CUDA(d->alloc(&d->text, n + 1));
    if (n) MHB_CUDA(cudaMemcpyAsync(d->text, text_h, n, cudaMemcpyHostToDevice, st));
    if (tables) {  // isalnum bitmap | lowercase keys | lowercase values
        if (tables->n_lower < 0 || !tables->alnum_bits || (tables->n_lower && (!tables->lower_keys || !tables->lower_vals)))
            return set_error(MHB_ERR_INVALID, "bad Unicode tables");
        const size_t words = 0x110000 / 32, nl = (size_t)tables->n_lower;
        const bool sig = tables->cased_bits && tables->ignorable_bits;
        // alnum | keys | vals | cased | ignorable
        MHB_CUDA(d->alloc(&d->tab_buf, words + nl * 4 + 2 * words + 1));
        uint32_t* tb = d->tab_buf;
        MHB_CUDA(cudaMemcpyAsync(tb, tables->alnum_bits, words * 4, cudaMemcpyHostToDevice, st));
        if (nl) {
            MHB_CUDA(cudaMemcpyAsync(tb + words, tables->lower_keys, nl * 4, cudaMemcpyHostToDevice, st));
            MHB_CUDA(cudaMemcpyAsync(tb + words + nl, tables->lower_vals, nl * 12, cudaMemcpyHostToDevice, st));
        }
        uint32_t* cased = tb + words + 4 * nl;
        if (sig) {
            MHB_CUDA(cudaMemcpyAsync(cased, tables->cased_bits, words * 4, cudaMemcpyHostToDevice, st));
            MHB_CUDA(cudaMemcpyAsync(cased + words, tables->ignorable_bits, words * 4, cudaMemcpyHostToDevice, st));
        }
        d->uni = true;
        d->tab = UniTab{tb, tb + words, tb + words + nl, (int)nl, sig ? cased : nullptr, sig ? cased + words : nullptr};
    }
    tm.mark("scan: H2D text");
    try {
        Scratch sc(st);
        // count the breaks, then select their positions
        thrust::counting_iterator<int64_t> iota(0);
        auto flags = thrust::make_transform_iterator(iota, BreakFlag{d->text});
        int64_t* n_brk_d = sc.get<int64_t>(1);
        size_t tb = 0;
        MHB_CUDA(cub::DeviceReduce::Sum(nullptr, tb, flags, n_brk_d, n, st));
        void* tmp = sc.get<char>(tb);
        MHB_CUDA(cub::DeviceReduce::Sum(tmp, tb, flags, n_brk_d, n, st));
        int64_t n_brk = 0;
        MHB_CUDA(cudaMemcpyAsync(&n_brk, n_brk_d, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        MHB_CUDA(cudaStreamSynchronize(st));
        int64_t* brk = sc.get<int64_t>(n_brk);
        int64_t* n_sel = sc.get<int64_t>(1);
        tb = 0;
        MHB_CUDA(cub::DeviceSelect::If(nullptr, tb, iota, brk, n_sel, n, IsBreak{d->text}, st));
        tmp = sc.get<char>(tb);
        MHB_CUDA(cub::DeviceSelect::If(tmp, tb, iota, brk, n_sel, n, IsBreak{d->text}, st));
        MHB_CUDA(d->alloc(&d->line_start, n_brk + 2));
        MHB_CUDA(d->alloc(&d->line_end, n_brk + 2));
        lines_from_breaks<<<blocks_for(n_brk + 1), 256, 0, st>>>(brk, n_brk, d->text, n, d->line_start, d->line_end);
        int64_t last_start = 0;
        MHB_CUDA(cudaMemcpyAsync(&last_start, d->line_start + n_brk, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        MHB_CUDA(cudaStreamSynchronize(st));
        tm.mark("scan: lines");
        d->n_docs = n_brk + (last_start < n ? 1 : 0);
        const int64_t nd = d->n_docs;
        MHB_CUDA(d->alloc(&d->count, nd + 1));
        MHB_CUDA(d->alloc(&d->deferred, nd));
        MHB_CUDA(d->alloc(&d->ucount, nd + 1));
        MHB_CUDA(d->alloc(&d->ubytes, nd + 1));
        MHB_CUDA(cudaMemsetAsync(d->count, 0, (nd + 1) * sizeof(int64_t), st));
        MHB_CUDA(cudaMemsetAsync(d->ucount, 0, (nd + 1) * sizeof(int64_t), st));
        MHB_CUDA(cudaMemsetAsync(d->ubytes, 0, (nd + 1) * sizeof(int64_t), st));
        if (nd) {
            scan_lines<<<warp_blocks(nd), 32 * kWarpsPerBlock, 0, st>>>(d->text, d->line_start, d->line_end, nd,
                                                                        d->count, d->deferred, d->uni);
            if (d->uni)
                uni_lines<false><<<blocks_for(nd, 128), 128, 0, st>>>(
                    d->text, d->line_start, d->line_end, nd, d->tab, d->deferred, d->ucount, d->ubytes, nullptr,
                    nullptr, 0, nullptr, nullptr, nullptr, nullptr);
        }
        line_start.resize(nd);
        line_end.resize(nd);
        d->deferred_h.resize(nd);
        if (nd) {
            MHB_CUDA(cudaMemcpyAsync(line_start.data(), d->line_start, nd * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaMemcpyAsync(line_end.data(), d->line_end, nd * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaMemcpyAsync(d->deferred_h.data(), d->deferred, nd, cudaMemcpyDeviceToHost, st));
        }
        MHB_CUDA(cudaStreamSynchronize(st));
        tm.mark("scan: tokens + D2H lines");
    } catch (const std::bad_alloc&) {
        return set_error(MHB_ERR_CUDA, "device allocation failed in corpus scan");
    }
    MHB_CUDA(cudaGetLastError());
    deferred_lines.clear();
    for (int64_t k = 0; k < d->n_docs; ++k)
        if (d->deferred_h[k] == 1) deferred_lines.push_back(k);
    *out = d.release();
    return MHB_OK;
}

int corpus_device_set_terms(CorpusDevice* d, int64_t n_lines, const int64_t* lines, const int64_t* line_ptr,
                            const char* blob, const int64_t* term_offsets) {
    if (d->interned) return set_error(MHB_ERR_INVALID, "corpus already interned");
    for (int64_t k = 0; k < n_lines; ++k) {
        const int64_t ln = lines[k];
        if (ln < 0 || ln >= d->n_docs || d->deferred_h[ln] != 1)
            return set_error(MHB_ERR_INVALID, "line %lld is not a deferred line awaiting terms", (long long)ln);
        const int64_t t0 = line_ptr[k], t1 = line_ptr[k + 1];
        if (t1 < t0) return set_error(MHB_ERR_INVALID, "bad term count for line %lld", (long long)ln);
        d->dl_line.push_back(ln);
        d->dl_cnt.push_back(t1 - t0);
        d->dl_first.push_back((int64_t)d->dterm_off.size() - 1);
        for (int64_t j = t0; j < t1; ++j) {
            const int64_t len = term_offsets[j + 1] - term_offsets[j];
            if (len <= 0 || len > 0xFFFFFFFFll) return set_error(MHB_ERR_INVALID, "bad term length");
            d->dblob.insert(d->dblob.end(), blob + term_offsets[j], blob + term_offsets[j] + len);
            d->dterm_off.push_back((int64_t)d->dblob.size());
        }
        d->deferred_h[ln] = 2;
    }
    return MHB_OK;
}

int corpus_device_intern(CorpusDevice* d, int64_t* nnz, int64_t* n_terms, int64_t* term_bytes,
                         int64_t* empty_docs) {
    for (int64_t k = 0; k < d->n_docs; ++k)
        if (d->deferred_h[k] == 1)
            return set_error(MHB_ERR_INVALID, "deferred line %lld has no terms yet (mhb_corpus_set_terms)",
                             (long long)k);
    if (!d->interned) {
        MHB_CUDA(cudaSetDevice(d->device));
        cudaStream_t st = d->st;
        const int64_t nd = d->n_docs;
        StageTimer tm(st);
        try {
            Scratch sc(st);
            // deferred lines: supplied term counts and the blob
            const int64_t ndl = (int64_t)d->dl_line.size();
            int64_t* dfirst = sc.get<int64_t>(nd + 1);
            int64_t* scount = sc.get<int64_t>(nd + 1);
            int64_t* count = sc.get<int64_t>(nd + 1);
            MHB_CUDA(cudaMemsetAsync(scount, 0, (nd + 1) * sizeof(int64_t), st));
            int64_t* dterm_off = sc.get<int64_t>(d->dterm_off.size());
            // blob region: caller-supplied terms, then the lowered bytes of device-tokenized Unicode lines
            int64_t* uoff = sc.get<int64_t>(nd + 1);
            size_t tbu = 0;
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tbu, d->ubytes, uoff, nd + 1, st));
            void* tmpu = sc.get<char>(tbu);
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(tmpu, tbu, d->ubytes, uoff, nd + 1, st));
            int64_t UB = 0;
            MHB_CUDA(cudaMemcpyAsync(&UB, uoff + nd, 8, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            const int64_t D = (int64_t)d->dblob.size();
            uint8_t* dblob = sc.get<uint8_t>(D + UB + 1);
            if (ndl) {
                int64_t* a = sc.get<int64_t>(ndl);
                int64_t* b = sc.get<int64_t>(ndl);
                int64_t* c = sc.get<int64_t>(ndl);
                MHB_CUDA(cudaMemcpyAsync(a, d->dl_line.data(), ndl * 8, cudaMemcpyHostToDevice, st));
                MHB_CUDA(cudaMemcpyAsync(b, d->dl_cnt.data(), ndl * 8, cudaMemcpyHostToDevice, st));
                MHB_CUDA(cudaMemcpyAsync(c, d->dl_first.data(), ndl * 8, cudaMemcpyHostToDevice, st));
                scatter_deferred<<<blocks_for(ndl), 256, 0, st>>>(a, b, c, ndl, scount, dfirst);
            }
            MHB_CUDA(cudaMemcpyAsync(dterm_off, d->dterm_off.data(), d->dterm_off.size() * 8, cudaMemcpyHostToDevice, st));
            if (!d->dblob.empty())
                MHB_CUDA(cudaMemcpyAsync(dblob, d->dblob.data(), d->dblob.size(), cudaMemcpyHostToDevice, st));
            const Src src{d->text, dblob, d->n_bytes};
            // token offsets per line
            int64_t* tok_off = sc.get<int64_t>(nd + 1);
            size_t tb = 0;
            add_counts<<<blocks_for(nd + 1), 256, 0, st>>>(d->count, scount, d->ucount, nd + 1, count);
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, count, tok_off, nd + 1, st));
            void* tmp = sc.get<char>(tb);
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, count, tok_off, nd + 1, st));
            int64_t T = 0;
            MHB_CUDA(cudaMemcpyAsync(&T, tok_off + nd, 8, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            tm.mark("intern: deferred + offsets");
            if (T >= (1ll << 31)) return set_error(MHB_ERR_UNSUPPORTED, "more than 2^31 tokens in one corpus call");
            int64_t* tok_start = sc.get<int64_t>(T);
            uint32_t* tok_len = sc.get<uint32_t>(T);
            uint32_t* tok_line = sc.get<uint32_t>(T);
            if (nd)
                write_tokens<<<warp_blocks(nd), 32 * kWarpsPerBlock, 0, st>>>(
                    d->text, d->n_bytes, d->line_start, d->line_end, nd, d->count, d->deferred, tok_off, dfirst,
                    dterm_off, tok_start, tok_len, tok_line);
            if (nd && d->uni)
                uni_lines<true><<<blocks_for(nd, 128), 128, 0, st>>>(
                    d->text, d->line_start, d->line_end, nd, d->tab, d->deferred, nullptr, nullptr, tok_off, uoff,
                    d->n_bytes + D, dblob + D, tok_start, tok_len, tok_line);
            // hash, sort, verify runs (re-hash with another seed on a collision)
            tm.mark("intern: write tokens");
            unsigned long long* h = sc.get<unsigned long long>(T);
            unsigned long long* key = sc.get<unsigned long long>(T);
            uint32_t* idx = sc.get<uint32_t>(T);
            unsigned long long* hs = sc.get<unsigned long long>(T);
            uint32_t* order = sc.get<uint32_t>(T);
            uint32_t* head = sc.get<uint32_t>(T);
            int* coll = sc.get<int>(1);
            const int Ti = (int)T;
            tb = 0;
            MHB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, h, hs, idx, order, Ti, 0, 64, st));
            void* sort_tmp = sc.get<char>(tb);
            size_t sort_tb = tb;
            int collided = 1;
            for (uint64_t seed = 0; seed < 4 && collided; ++seed) {
                hash_tokens<<<blocks_for(T), 256, 0, st>>>(src, tok_start, tok_len, T, seed * 0x632BE59BD9B4E019ull, h,
                                                          key, idx);
                tb = sort_tb;
                MHB_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, tb, h, hs, idx, order, Ti, 0, 64, st));
                MHB_CUDA(cudaMemsetAsync(coll, 0, sizeof(int), st));
                run_heads<<<blocks_for(T), 256, 0, st>>>(src, hs, order, tok_start, tok_len, T, head, coll);
                MHB_CUDA(cudaMemcpyAsync(&collided, coll, sizeof(int), cudaMemcpyDeviceToHost, st));
                MHB_CUDA(cudaStreamSynchronize(st));
            }
            if (collided) return set_error(MHB_ERR_UNSUPPORTED, "64-bit term hash collided under 4 seeds");
            tm.mark("intern: hash+sort+verify");
            // runs = distinct terms
            uint32_t* run_incl = sc.get<uint32_t>(T);
            tb = 0;
            MHB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head, run_incl, Ti, st));
            tmp = sc.get<char>(tb);
            MHB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, head, run_incl, Ti, st));
            uint32_t U32 = 0;
            if (T) MHB_CUDA(cudaMemcpyAsync(&U32, run_incl + T - 1, 4, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            const int64_t U = T ? U32 : 0;
            uint32_t* run_of_tok = sc.get<uint32_t>(T);
            uint32_t* run_tok = sc.get<uint32_t>(U);
            uint32_t* run_line = sc.get<uint32_t>(U);
            unsigned long long* run_key = sc.get<unsigned long long>(U);
            uint32_t* run_idx = sc.get<uint32_t>(U);
            run_info<<<blocks_for(T), 256, 0, st>>>(head, run_incl, order, tok_line, key, T, run_of_tok, run_tok,
                                                    run_line, run_key, run_idx);
            // vocabulary order: (first line, term bytes)
            unsigned long long* key_s = sc.get<unsigned long long>(U);
            uint32_t* ord1 = sc.get<uint32_t>(U);
            uint32_t* line1 = sc.get<uint32_t>(U);
            uint32_t* line_s = sc.get<uint32_t>(U);
            uint32_t* ord2 = sc.get<uint32_t>(U);
            const int Ui = (int)U;
            tb = 0;
            MHB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, run_key, key_s, run_idx, ord1, Ui, 0, 64, st));
            size_t tb2 = 0;
            MHB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, line1, line_s, ord1, ord2, Ui, 0, 32, st));
            tmp = sc.get<char>(std::max(tb, tb2));
            MHB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, run_key, key_s, run_idx, ord1, Ui, 0, 64, st));
            gather_u32<<<blocks_for(U), 256, 0, st>>>(run_line, ord1, U, line1);
            tb2 = std::max(tb, tb2);
            MHB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb2, line1, line_s, ord1, ord2, Ui, 0, 32, st));
            fix_ties<<<blocks_for(U), 256, 0, st>>>(src, ord2, run_line, run_key, run_tok, tok_start, tok_len, U);
            uint32_t* id_of_run = sc.get<uint32_t>(U);
            int64_t* term_len = sc.get<int64_t>(U + 1);
            assign_ids<<<blocks_for(U + 1), 256, 0, st>>>(ord2, run_tok, tok_len, U, id_of_run, term_len);
            MHB_CUDA(d->alloc(&d->voff, U + 1));
            tb = 0;
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, term_len, d->voff, U + 1, st));
            tmp = sc.get<char>(tb);
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, term_len, d->voff, U + 1, st));
            int64_t vbytes = 0;
            MHB_CUDA(cudaMemcpyAsync(&vbytes, d->voff + U, 8, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            tm.mark("intern: runs + vocab order");
            MHB_CUDA(d->alloc(&d->vblob, vbytes + 1));
            write_vocab<<<blocks_for(U), 256, 0, st>>>(src, ord2, run_tok, tok_start, tok_len, d->voff, U, d->vblob);
            // documents: ids per token, sorted within each line, unique -> CSR
            uint32_t* tid = sc.get<uint32_t>(T);
            uint32_t* tid_s = sc.get<uint32_t>(T);
            token_ids<<<blocks_for(T), 256, 0, st>>>(run_of_tok, id_of_run, T, tid);
            tb = 0;
            MHB_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, tid, tid_s, Ti, (int)nd, tok_off, tok_off + 1,
                                                        st));
            tmp = sc.get<char>(tb);
            MHB_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, tb, tid, tid_s, Ti, (int)nd, tok_off, tok_off + 1, st));
            tm.mark("intern: vocab + seg sort");
            int64_t* keep = sc.get<int64_t>(T + 1);
            int64_t* pos = sc.get<int64_t>(T + 1);
            unique_flags<<<blocks_for(T + 1), 256, 0, st>>>(tid_s, tok_line, tok_off, T, keep);
            tb = 0;
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, pos, T + 1, st));
            tmp = sc.get<char>(tb);
            MHB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, keep, pos, T + 1, st));
            int64_t kept = 0;
            MHB_CUDA(cudaMemcpyAsync(&kept, pos + T, 8, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            MHB_CUDA(d->alloc(&d->ids, kept));
            MHB_CUDA(d->alloc(&d->indptr, nd + 1));
            unsigned long long* empty = sc.get<unsigned long long>(1);
            MHB_CUDA(cudaMemsetAsync(empty, 0, 8, st));
            compact_csr<<<blocks_for(std::max(T, nd + 1)), 256, 0, st>>>(tid_s, keep, pos, tok_off, T, nd, d->ids,
                                                                         d->indptr, empty);
            unsigned long long empty_h = 0;
            MHB_CUDA(cudaMemcpyAsync(&empty_h, empty, 8, cudaMemcpyDeviceToHost, st));
            MHB_CUDA(cudaStreamSynchronize(st));
            MHB_CUDA(cudaGetLastError());
            tm.mark("intern: unique + CSR");
            d->nnz = kept;
            d->n_terms = U;
            d->term_bytes = vbytes;
            d->empty = (int64_t)empty_h;
            d->interned = true;
        } catch (const std::bad_alloc&) {
            return set_error(MHB_ERR_CUDA, "device allocation failed in corpus intern");
        }
        MHB_CUDA(cudaStreamSynchronize(d->st));
    }
    if (nnz) *nnz = d->nnz;
    if (n_terms) *n_terms = d->n_terms;
    if (term_bytes) *term_bytes = d->term_bytes;
    if (empty_docs) *empty_docs = d->empty;
    return MHB_OK;
}

int corpus_device_export(const CorpusDevice* d, int64_t* indptr, uint32_t* ids, int64_t* term_offsets,
                         char* term_blob) {
    if (!d->interned) return set_error(MHB_ERR_INVALID, "call mhb_corpus_intern first");
    MHB_CUDA(cudaSetDevice(d->device));
    cudaStream_t st = d->st;
    if (indptr) MHB_CUDA(cudaMemcpyAsync(indptr, d->indptr, (d->n_docs + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (ids && d->nnz) MHB_CUDA(cudaMemcpyAsync(ids, d->ids, d->nnz * 4, cudaMemcpyDeviceToHost, st));
    if (term_offsets) MHB_CUDA(cudaMemcpyAsync(term_offsets, d->voff, (d->n_terms + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (term_blob && d->term_bytes)
        MHB_CUDA(cudaMemcpyAsync(term_blob, d->vblob, d->term_bytes, cudaMemcpyDeviceToHost, st));
    MHB_CUDA(cudaStreamSynchronize(st));
    return MHB_OK;
}

int corpus_device_export_device(const CorpusDevice* d, int64_t* indptr, uint32_t* ids, void* stream) {
    if (!d->interned) return set_error(MHB_ERR_INVALID, "call mhb_corpus_intern first");
    MHB_CUDA(cudaSetDevice(d->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (indptr) MHB_CUDA(cudaMemcpyAsync(indptr, d->indptr, (d->n_docs + 1) * 8, cudaMemcpyDeviceToDevice, st));
    if (ids && d->nnz) MHB_CUDA(cudaMemcpyAsync(ids, d->ids, d->nnz * 4, cudaMemcpyDeviceToDevice, st));
    return MHB_OK;
}

void corpus_device_free(CorpusDevice* d) { delete d; }

}  // namespace mhb
