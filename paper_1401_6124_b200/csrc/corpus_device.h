// corpus_device.h -- device (B200) backend of the corpus ingest (corpus_gpu.cu),
// driven through the same mhb_corpus_* C ABI as the host backend (corpus.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "mhb.h"

namespace mhb {

struct CorpusDevice;  // device buffers + results of one ingest

// Lines + per-line token counts + non-ASCII detection on the GPU.  Fills the host
// line arrays and the list of deferred (non-ASCII) lines.  Synchronous.
int corpus_device_scan(const char* text, int64_t n_bytes, int device, const mhb_unicode_tables* tables,
                       CorpusDevice** out,
                       std::vector<int64_t>& line_start, std::vector<int64_t>& line_end,
                       std::vector<int64_t>& deferred_lines);
int corpus_device_set_terms(CorpusDevice* d, int64_t n_lines, const int64_t* lines, const int64_t* line_ptr,
                            const char* blob, const int64_t* term_offsets);
int corpus_device_intern(CorpusDevice* d, int64_t* nnz, int64_t* n_terms, int64_t* term_bytes,
                         int64_t* empty_docs);
int corpus_device_export(const CorpusDevice* d, int64_t* indptr, uint32_t* ids, int64_t* term_offsets,
                         char* term_blob);
int corpus_device_export_device(const CorpusDevice* d, int64_t* indptr, uint32_t* ids, void* stream);
void corpus_device_free(CorpusDevice* d);

}  // namespace mhb
