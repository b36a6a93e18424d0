// corpus.cpp -- native corpus ingest: one document per line -> CSR feature ids.
//
// Restates minhashlab.corpus.build_corpus / tokenize / Vocabulary
// (reference src/corpus.py:18-80) for the step before the signing path:
//   * lines: Python text-mode iteration with universal newlines -- a line ends at
//     "\n", "\r\n" or a lone "\r"; a final line without terminator still counts;
//   * tokenize: lowercase, maximal runs of [^\W_] (alphanumerics), deduplicate, sort;
//   * vocabulary ids in first-occurrence order over (document order, sorted terms
//     of the document) -- Vocabulary.add called in that order;
//   * each document is the sorted id set (FeatureSet = np.unique).
// Pure-ASCII lines are tokenized here (ASCII [^\W_] is [A-Za-z0-9], ASCII lower()
// maps only A-Z).  Lines with a byte >= 0x80 need Unicode tables (Python's
// str.lower / str.isalnum); they are "deferred": the caller tokenizes them with the
// reference's own rules and hands the sorted UTF-8 terms back (UTF-8 byte order is
// code-point order, the order of Python's sorted()).
//
// Parallel plan (std::thread, T workers, lines split into T contiguous byte-balanced
// parts; deferred lines form part T):
//   scan    each worker tokenizes its lines and interns every term into its own
//           table (term -> dense entry holding the entry's first occurrence
//           (line, rank)); a document is kept as 4-byte entry indices;
//   merge   S = T hash shards; shard s walks every part's entries whose hash falls
//           in s, inserts them into its global table keeping the smallest first
//           occurrence, and records the global entry of each local entry;
//   ids     vocabulary id = rank of a term's first ordinal (ordinal = number of terms
//           in the documents before its line + its rank in the line): a bitmap over
//           ordinals + prefix popcounts;
//   export  documents map entry -> id and sort.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string_view>
#include <thread>
#include <vector>

#include "common.h"
#include "corpus_device.h"

namespace {

using std::string_view;

inline uint64_t hash_bytes(const char* p, size_t n) {
    // multiply-xorshift over 8-byte words (not cryptographic; equality is always
    // confirmed on the bytes)
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (n * 0xFF51AFD7ED558CCDull);
    while (n >= 8) {
        uint64_t w;
        std::memcpy(&w, p, 8);
        h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
        h ^= h >> 29;
        p += 8;
        n -= 8;
    }
    uint64_t w = 0;
    std::memcpy(&w, p, n);
    h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 32;
    h *= 0xFF51AFD7ED558CCDull;
    return h ^ (h >> 29);
}

// Chunked byte arena: stable pointers for lowercased / caller-supplied terms.
struct Arena {
    std::vector<std::unique_ptr<char[]>> blocks;
    size_t used = 0, cap = 0;
    char* alloc(size_t n) {
        if (used + n > cap) {
            cap = std::max<size_t>(n, 1 << 20);
            blocks.emplace_back(new char[cap]);
            used = 0;
        }
        char* r = blocks.back().get() + used;
        used += n;
        return r;
    }
};

struct Tok {  // a term of the line being tokenized
    const char* p;
    uint64_t key;  // first 8 bytes, big-endian, zero-padded (sort prefix)
    uint32_t len;
};

inline uint64_t prefix_key(const char* p, uint32_t n) {
    uint64_t w = 0;
    std::memcpy(&w, p, n < 8 ? n : 8);
    return __builtin_bswap64(w);
}

// Byte order of the terms (= Python's code-point order for UTF-8).  Terms hold no
// NUL bytes, so the zero padding of the prefix key orders a proper prefix first.
inline bool tok_less(const Tok& a, const Tok& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.len <= 8 || b.len <= 8) return a.len < b.len;
    return string_view(a.p + 8, a.len - 8) < string_view(b.p + 8, b.len - 8);
}
inline bool tok_eq(const Tok& a, const Tok& b) {
    return a.key == b.key && a.len == b.len && (a.len <= 8 || std::memcmp(a.p + 8, b.p + 8, a.len - 8) == 0);
}

// byte classes: 0 separator, 1 [a-z0-9], 2 [A-Z], 4 non-ASCII
struct ByteClass {
    uint8_t c[256];
    constexpr ByteClass() : c() {
        for (int b = 0; b < 256; ++b)
            c[b] = b >= 0x80 ? 4 : ((b >= 'a' && b <= 'z') || (b >= '0' && b <= '9')) ? 1 : (b >= 'A' && b <= 'Z') ? 2 : 0;
    }
};
constexpr ByteClass kClass{};

constexpr int kRankBits = 24;  // first occurrence packed as line << 24 | rank

struct Entry {
    const char* p;
    uint64_t h;
    uint64_t key;    // prefix key (as Tok)
    uint64_t first;  // packed (line, rank); in a global table, the id once assigned
    uint32_t len;
};

// Open addressing over dense entries (entry indices stay valid when the table grows).
// A slot carries the prefix key and length, so terms of <= 8 bytes are matched
// without touching the entry or the term bytes.
struct Table {
    struct Slot {
        uint64_t key;
        uint32_t len;
        uint32_t idx1;  // entry index + 1, 0 = empty
    };
    std::vector<Entry> ent;
    std::vector<Slot> slot;
    size_t mask = 0;
    void init(size_t expect) {
        size_t c = 64;
        while (c < expect * 2) c <<= 1;
        slot.assign(c, Slot{0, 0, 0});
        mask = c - 1;
        ent.clear();
        ent.reserve(expect);
    }
    void grow() {
        slot.assign(slot.size() * 2, Slot{0, 0, 0});
        mask = slot.size() - 1;
        for (size_t e = 0; e < ent.size(); ++e) {
            size_t i = ent[e].h & mask;
            while (slot[i].idx1) i = (i + 1) & mask;
            slot[i] = Slot{ent[e].key, ent[e].len, (uint32_t)(e + 1)};
        }
    }
    // index of the term's entry, inserting it with `first` if absent
    uint32_t intern(const char* p, uint32_t len, uint64_t h, uint64_t key, uint64_t first) {
        if ((ent.size() + 1) * 4 > slot.size() * 3) grow();
        size_t i = h & mask;
        for (;;) {
            const Slot s = slot[i];
            if (!s.idx1) {
                ent.push_back(Entry{p, h, key, first, len});
                slot[i] = Slot{key, len, (uint32_t)ent.size()};
                return (uint32_t)(ent.size() - 1);
            }
            if (s.key == key && s.len == len) {
                if (len <= 8) return s.idx1 - 1;
                const Entry& e = ent[s.idx1 - 1];
                if (e.h == h && std::memcmp(e.p + 8, p + 8, len - 8) == 0) return s.idx1 - 1;
            }
            i = (i + 1) & mask;
        }
    }
};

template <typename F>
void parallel_for(int T, F&& f) {
    if (T == 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(t); });
    for (auto& x : th) x.join();
}

// shard from the high hash bits (table slots use the low bits)
inline int shard_of(uint64_t h, int S) { return (int)(((h >> 32) * (uint64_t)S) >> 32); }

}  // namespace

struct mhb_corpus {
    const char* text = nullptr;
    int64_t n_bytes = 0;
    int T = 1;
    std::vector<int64_t> line_start, line_end;     // [n_docs]
    std::vector<uint8_t> deferred;                 // [n_docs]: 0 native, 1 awaiting terms, 2 supplied
    std::vector<int64_t> deferred_lines;
    std::vector<int64_t> range;                    // part line ranges [T+1]
    std::vector<int64_t> term_off;                 // [n_docs]: offset into its part's doc_terms
    std::vector<int64_t> term_cnt;                 // [n_docs]
    // parts 0..T-1: the native lines of range t; part T: the deferred lines
    std::vector<Table> local;                      // [T+1]
    std::vector<std::vector<uint32_t>> doc_terms;  // [T+1]: entry indices, line by line
    std::vector<Arena> arenas;                     // [T+1]
    // interned
    bool interned = false;
    std::vector<int64_t> indptr;
    std::vector<uint32_t> ids;
    std::vector<Table> global;                     // [S]
    std::vector<const Entry*> vocab;               // by id
    int64_t vocab_bytes = 0, empty_docs = 0;
    // device backend (corpus_gpu.cu); null for the host backend
    mhb::CorpusDevice* dev = nullptr;
    ~mhb_corpus() {
        if (dev) mhb::corpus_device_free(dev);
    }
};

namespace {

void split_lines(mhb_corpus* c) {
    const char* s = c->text;
    const int64_t n = c->n_bytes;
    const int T = c->T;
    // break positions per byte range: '\r', or '\n' not preceded by '\r'
    std::vector<std::vector<int64_t>> brk(T);
    parallel_for(T, [&](int t) {
        const int64_t lo = n * t / T, hi = n * (t + 1) / T;
        auto& b = brk[t];
        b.reserve((hi - lo) / 64 + 16);
        for (int64_t j = lo; j < hi; ++j) {
            const char ch = s[j];
            if (ch == '\r' || (ch == '\n' && !(j > 0 && s[j - 1] == '\r'))) b.push_back(j);
        }
    });
    size_t nb = 0;
    for (auto& b : brk) nb += b.size();
    c->line_start.reserve(nb + 1);
    c->line_end.reserve(nb + 1);
    int64_t start = 0;
    for (auto& b : brk)
        for (int64_t j : b) {
            c->line_start.push_back(start);
            c->line_end.push_back(j);
            start = j + ((s[j] == '\r' && j + 1 < n && s[j + 1] == '\n') ? 2 : 1);
        }
    if (start < n) {  // last line without terminator
        c->line_start.push_back(start);
        c->line_end.push_back(n);
    }
}

// Native tokens of one line into `toks` (sorted, unique): the maximal ASCII
// alphanumeric runs whose segment (maximal run of [A-Za-z0-9\x80-\xff]) is pure
// ASCII.  *foreign: the line holds a byte >= 0x80 (its other segments are the
// caller's, see mhb_corpus_set_terms).  A line holding U+03A3 (bytes CE A3, Python's
// only context-dependent lowercase) has no native tokens.
void tokenize_native(const unsigned char* p, int64_t len, Arena& ar, std::vector<Tok>& toks, bool* foreign) {
    toks.clear();
    *foreign = false;
    bool sigma = false;
    for (int64_t j = 0; j < len;) {
        const uint8_t cj = kClass.c[p[j]];
        if (cj == 0) {
            ++j;
            continue;
        }
        int64_t k = j;
        uint8_t up = 0, ck;
        while (k < len && ((ck = kClass.c[p[k]]) & 3)) {
            up |= ck;
            ++k;
        }
        if (k < len && (kClass.c[p[k]] & 4)) {  // the segment holds non-ASCII bytes: not native
            *foreign = true;
            while (k < len && kClass.c[p[k]] != 0) {
                sigma |= p[k] == 0xCE && k + 1 < len && p[k + 1] == 0xA3;
                ++k;
            }
            j = k;
            continue;
        }
        const char* tp = reinterpret_cast<const char*>(p + j);
        const uint32_t n = (uint32_t)(k - j);
        if (up & 2) {
            char* q = ar.alloc(n);
            for (uint32_t m = 0; m < n; ++m) q[m] = (char)(tp[m] | (kClass.c[(uint8_t)tp[m]] == 2 ? 0x20 : 0));
            tp = q;
        }
        toks.push_back(Tok{tp, prefix_key(tp, n), n});
        j = k;
    }
    if (sigma) toks.clear();
    std::sort(toks.begin(), toks.end(), tok_less);
    toks.erase(std::unique(toks.begin(), toks.end(), tok_eq), toks.end());
}

void scan_parts(mhb_corpus* c) {
    const int64_t n_docs = (int64_t)c->line_start.size();
    const int T = c->T;
    c->deferred.assign(n_docs, 0);
    c->term_off.assign(n_docs, 0);
    c->term_cnt.assign(n_docs, 0);
    c->range.assign(T + 1, n_docs);
    c->range[0] = 0;
    for (int t = 1; t < T; ++t) {
        const int64_t target = c->n_bytes * t / T;
        c->range[t] = std::lower_bound(c->line_start.begin(), c->line_start.end(), target) - c->line_start.begin();
    }
    for (int t = 1; t <= T; ++t) c->range[t] = std::max(c->range[t], c->range[t - 1]);
    c->local.resize(T + 1);
    c->doc_terms.resize(T + 1);
    c->arenas.resize(T + 1);
    std::vector<int> too_many(T, 0);
    parallel_for(T, [&](int t) {
        const int64_t d0 = c->range[t], d1 = c->range[t + 1];
        const int64_t bytes = d1 > d0 ? c->line_end[d1 - 1] - c->line_start[d0] : 0;
        Table& tab = c->local[t];
        tab.init(4096);
        auto& dt = c->doc_terms[t];
        dt.reserve(bytes / 8 + 16);
        std::vector<Tok> toks;
        for (int64_t d = d0; d < d1; ++d) {
            const unsigned char* p = reinterpret_cast<const unsigned char*>(c->text + c->line_start[d]);
            bool foreign;
            tokenize_native(p, c->line_end[d] - c->line_start[d], c->arenas[t], toks, &foreign);
            if (foreign) {  // interned in mhb_corpus_set_terms, with the caller's terms
                c->deferred[d] = 1;
                continue;
            }
            if (toks.size() >= (1u << kRankBits)) too_many[t] = 1;
            c->term_off[d] = (int64_t)dt.size();
            c->term_cnt[d] = (int64_t)toks.size();
            for (size_t r = 0; r < toks.size(); ++r) {
                const Tok& k = toks[r];
                dt.push_back(tab.intern(k.p, k.len, hash_bytes(k.p, k.len), k.key, ((uint64_t)d << kRankBits) | r));
            }
        }
    });
    for (int t = 0; t < T; ++t)
        if (too_many[t]) throw std::length_error("a document holds 2^24 or more distinct terms");
    for (int64_t d = 0; d < n_docs; ++d)
        if (c->deferred[d]) c->deferred_lines.push_back(d);
    c->local[T].init(1024);
}

}  // namespace

extern "C" int mhb_corpus_scan(const char* text, int64_t n_bytes, int32_t n_threads, mhb_corpus** out) {
    using namespace mhb;
    clear_error();
    if (!out || n_bytes < 0 || (n_bytes > 0 && !text)) return set_error(MHB_ERR_INVALID, "bad corpus buffer");
    *out = nullptr;
    try {
        auto c = std::make_unique<mhb_corpus>();
        c->text = text;
        c->n_bytes = n_bytes;
        int T = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
        T = std::max(1, std::min(T, 256));
        if (n_bytes < (int64_t)T * (1 << 16)) T = std::max<int>(1, (int)(n_bytes >> 16));  // >= 64 KiB per part
        c->T = T;
        split_lines(c.get());
        scan_parts(c.get());
        *out = c.release();
        return MHB_OK;
    } catch (const std::exception& e) {
        return set_error(MHB_ERR_INVALID, "corpus scan failed: %s", e.what());
    }
}

extern "C" int mhb_corpus_scan_device(const char* text, int64_t n_bytes, int32_t device,
                                      const mhb_unicode_tables* tables, mhb_corpus** out) {
    using namespace mhb;
    clear_error();
    if (!out || n_bytes < 0 || (n_bytes > 0 && !text)) return set_error(MHB_ERR_INVALID, "bad corpus buffer");
    *out = nullptr;
    try {
        auto c = std::make_unique<mhb_corpus>();
        c->text = text;
        c->n_bytes = n_bytes;
        const int rc = corpus_device_scan(text, n_bytes, device, tables, &c->dev, c->line_start, c->line_end,
                                          c->deferred_lines);
        if (rc) return rc;
        *out = c.release();
        return MHB_OK;
    } catch (const std::exception& e) {
        return set_error(MHB_ERR_INVALID, "corpus scan failed: %s", e.what());
    }
}

extern "C" int mhb_corpus_info(const mhb_corpus* c, int64_t* n_docs, int64_t* n_deferred) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    if (n_docs) *n_docs = (int64_t)c->line_start.size();
    if (n_deferred) *n_deferred = (int64_t)c->deferred_lines.size();
    return MHB_OK;
}

extern "C" int mhb_corpus_deferred(const mhb_corpus* c, int64_t* lines, int64_t* starts, int64_t* lens) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    for (size_t k = 0; k < c->deferred_lines.size(); ++k) {
        const int64_t d = c->deferred_lines[k];
        if (lines) lines[k] = d;
        if (starts) starts[k] = c->line_start[d];
        if (lens) lens[k] = c->line_end[d] - c->line_start[d];
    }
    return MHB_OK;
}

extern "C" int mhb_corpus_set_terms(mhb_corpus* c, int64_t n_lines, const int64_t* lines, const int64_t* line_ptr,
                                    const char* blob, const int64_t* term_offsets) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    if (n_lines < 0 || (n_lines > 0 && (!lines || !line_ptr || !term_offsets)))
        return set_error(MHB_ERR_INVALID, "bad deferred-term arrays");
    if (c->dev) return corpus_device_set_terms(c->dev, n_lines, lines, line_ptr, blob, term_offsets);
    if (c->interned) return set_error(MHB_ERR_INVALID, "corpus already interned");
    const int64_t n_docs = (int64_t)c->line_start.size();
    const int P = c->T;  // the deferred part
    Table& tab = c->local[P];
    auto& dt = c->doc_terms[P];
    Arena& ar = c->arenas[P];
    std::vector<Tok> toks;
    for (int64_t k = 0; k < n_lines; ++k) {
        const int64_t d = lines[k];
        if (d < 0 || d >= n_docs || c->deferred[d] != 1)
            return set_error(MHB_ERR_INVALID, "line %lld is not a deferred line awaiting terms", (long long)d);
        const int64_t t0 = line_ptr[k], t1 = line_ptr[k + 1];
        if (t1 < t0) return set_error(MHB_ERR_INVALID, "bad term count for line %lld", (long long)d);
        // the line's native tokens + the supplied terms, sorted and deduplicated
        bool foreign;
        const unsigned char* p = reinterpret_cast<const unsigned char*>(c->text + c->line_start[d]);
        tokenize_native(p, c->line_end[d] - c->line_start[d], ar, toks, &foreign);
        for (int64_t j = t0; j < t1; ++j) {
            const int64_t len = term_offsets[j + 1] - term_offsets[j];
            if (len <= 0 || len > 0xFFFFFFFFll) return set_error(MHB_ERR_INVALID, "bad term length");
            char* q = ar.alloc(len);
            std::memcpy(q, blob + term_offsets[j], len);
            toks.push_back(Tok{q, prefix_key(q, (uint32_t)len), (uint32_t)len});
        }
        std::sort(toks.begin(), toks.end(), tok_less);
        toks.erase(std::unique(toks.begin(), toks.end(), tok_eq), toks.end());
        if (toks.size() >= (1u << kRankBits))
            return set_error(MHB_ERR_INVALID, "line %lld holds 2^24 or more distinct terms", (long long)d);
        c->term_off[d] = (int64_t)dt.size();
        c->term_cnt[d] = (int64_t)toks.size();
        for (size_t r = 0; r < toks.size(); ++r)
            dt.push_back(tab.intern(toks[r].p, toks[r].len, hash_bytes(toks[r].p, toks[r].len), toks[r].key,
                                    ((uint64_t)d << kRankBits) | r));
        c->deferred[d] = 2;
    }
    return MHB_OK;
}

extern "C" int mhb_corpus_intern(mhb_corpus* c, int64_t* nnz, int64_t* n_terms, int64_t* term_bytes,
                                 int64_t* empty_docs) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    if (c->dev) return corpus_device_intern(c->dev, nnz, n_terms, term_bytes, empty_docs);
    const int64_t n_docs = (int64_t)c->line_start.size();
    for (int64_t d : c->deferred_lines)
        if (c->deferred[d] != 2)
            return set_error(MHB_ERR_INVALID, "deferred line %lld has no terms yet (mhb_corpus_set_terms)",
                             (long long)d);
    try {
        if (!c->interned) {
            const int T = c->T, P = T + 1, S = T;
            // ordinal of each document's first term, in document order
            std::vector<int64_t> ord0(n_docs + 1, 0);
            for (int64_t d = 0; d < n_docs; ++d) ord0[d + 1] = ord0[d] + c->term_cnt[d];
            const int64_t total = ord0[n_docs];
            auto ordinal = [&](uint64_t packed) {
                return (uint64_t)ord0[packed >> kRankBits] + (packed & ((1ull << kRankBits) - 1));
            };
            // merge: shard s owns the terms whose hash maps to s
            std::vector<std::vector<uint32_t>> gidx(P);  // per part: local entry -> global entry
            for (int q = 0; q < P; ++q) gidx[q].resize(c->local[q].ent.size());
            c->global.resize(S);
            parallel_for(S, [&](int s) {
                size_t expect = 0;
                for (int q = 0; q < P; ++q) expect += c->local[q].ent.size() / S + 1;
                Table& g = c->global[s];
                g.init(expect);
                for (int q = 0; q < P; ++q) {
                    const auto& ent = c->local[q].ent;
                    for (size_t e = 0; e < ent.size(); ++e) {
                        if (shard_of(ent[e].h, S) != s) continue;
                        const uint32_t gi = g.intern(ent[e].p, ent[e].len, ent[e].h, ent[e].key, ent[e].first);
                        // the deferred part is not in document order: keep the smallest
                        if (ent[e].first < g.ent[gi].first) g.ent[gi].first = ent[e].first;
                        gidx[q][e] = gi;
                    }
                }
            });
            // ids: rank of each term's first ordinal
            const int64_t words = total / 64 + 1;
            std::unique_ptr<std::atomic<uint64_t>[]> bits(new std::atomic<uint64_t>[words]);
            parallel_for(T, [&](int t) {
                for (int64_t w = words * t / T; w < words * (t + 1) / T; ++w)
                    bits[w].store(0, std::memory_order_relaxed);
            });
            parallel_for(S, [&](int s) {
                for (const Entry& e : c->global[s].ent) {
                    const uint64_t o = ordinal(e.first);
                    bits[o >> 6].fetch_or(1ull << (o & 63), std::memory_order_relaxed);
                }
            });
            std::vector<int64_t> pre(words, 0), blk(T + 1, 0);
            parallel_for(T, [&](int t) {
                int64_t acc = 0;
                for (int64_t w = words * t / T; w < words * (t + 1) / T; ++w)
                    acc += __builtin_popcountll(bits[w].load(std::memory_order_relaxed));
                blk[t + 1] = acc;
            });
            for (int t = 0; t < T; ++t) blk[t + 1] += blk[t];
            parallel_for(T, [&](int t) {
                int64_t acc = blk[t];
                for (int64_t w = words * t / T; w < words * (t + 1) / T; ++w) {
                    pre[w] = acc;
                    acc += __builtin_popcountll(bits[w].load(std::memory_order_relaxed));
                }
            });
            const int64_t U = blk[T];
            if (U > 0xFFFFFFFFll) return set_error(MHB_ERR_UNSUPPORTED, "vocabulary exceeds 2^32 terms");
            c->vocab.assign(U, nullptr);
            std::vector<int64_t> vb(S, 0);
            parallel_for(S, [&](int s) {
                for (Entry& e : c->global[s].ent) {
                    const uint64_t o = ordinal(e.first);
                    const uint64_t below = bits[o >> 6].load(std::memory_order_relaxed) & ((1ull << (o & 63)) - 1);
                    e.first = (uint64_t)(pre[o >> 6] + __builtin_popcountll(below));  // now the id
                    c->vocab[e.first] = &e;
                    vb[s] += e.len + 1;  // + the '\n' separator of the export
                }
            });
            c->vocab_bytes = 0;
            for (int s = 0; s < S; ++s) c->vocab_bytes += vb[s];
            // local entry -> id
            std::vector<std::vector<uint32_t>> lid(P);
            parallel_for(P, [&](int q) {
                const auto& ent = c->local[q].ent;
                lid[q].resize(ent.size());
                for (size_t e = 0; e < ent.size(); ++e)
                    lid[q][e] = (uint32_t)c->global[shard_of(ent[e].h, S)].ent[gidx[q][e]].first;
            });
            // documents -> sorted id sets (CSR)
            c->indptr.assign(ord0.begin(), ord0.end());
            c->ids.resize(total);
            std::vector<int64_t> empties(T, 0);
            parallel_for(T, [&](int t) {
                for (int64_t d = c->range[t]; d < c->range[t + 1]; ++d) {
                    const int q = c->deferred[d] ? T : t;
                    uint32_t* o = c->ids.data() + ord0[d];
                    const int64_t cnt = c->term_cnt[d];
                    if (cnt == 0) ++empties[t];
                    const uint32_t* src = c->doc_terms[q].data() + c->term_off[d];
                    for (int64_t r = 0; r < cnt; ++r) o[r] = lid[q][src[r]];
                    std::sort(o, o + cnt);
                }
            });
            c->empty_docs = 0;
            for (int t = 0; t < T; ++t) c->empty_docs += empties[t];
            c->interned = true;
        }
        if (nnz) *nnz = (int64_t)c->ids.size();
        if (n_terms) *n_terms = (int64_t)c->vocab.size();
        if (term_bytes) *term_bytes = c->vocab_bytes;
        if (empty_docs) *empty_docs = c->empty_docs;
        return MHB_OK;
    } catch (const std::exception& e) {
        return set_error(MHB_ERR_INVALID, "corpus intern failed: %s", e.what());
    }
}

extern "C" int mhb_corpus_export(const mhb_corpus* c, int64_t* indptr, uint32_t* ids, int64_t* term_offsets,
                                 char* term_blob) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    if (c->dev) return corpus_device_export(c->dev, indptr, ids, term_offsets, term_blob);
    if (!c->interned) return set_error(MHB_ERR_INVALID, "call mhb_corpus_intern first");
    if (indptr) std::memcpy(indptr, c->indptr.data(), c->indptr.size() * sizeof(int64_t));
    if (ids && !c->ids.empty()) std::memcpy(ids, c->ids.data(), c->ids.size() * sizeof(uint32_t));
    if (term_offsets || term_blob) {
        int64_t off = 0;
        for (size_t v = 0; v < c->vocab.size(); ++v) {
            if (term_offsets) term_offsets[v] = off;
            if (term_blob) {
                std::memcpy(term_blob + off, c->vocab[v]->p, c->vocab[v]->len);
                term_blob[off + c->vocab[v]->len] = '\n';
            }
            off += c->vocab[v]->len + 1;
        }
        if (term_offsets) term_offsets[c->vocab.size()] = off;
    }
    return MHB_OK;
}

extern "C" int mhb_corpus_export_device(const mhb_corpus* c, int64_t* indptr, uint32_t* ids, void* stream) {
    using namespace mhb;
    clear_error();
    if (!c) return set_error(MHB_ERR_INVALID, "null corpus handle");
    if (!c->dev) return set_error(MHB_ERR_INVALID, "mhb_corpus_export_device needs a handle from mhb_corpus_scan_device");
    return corpus_device_export_device(c->dev, indptr, ids, stream);
}

extern "C" void mhb_corpus_free(mhb_corpus* c) { delete c; }
