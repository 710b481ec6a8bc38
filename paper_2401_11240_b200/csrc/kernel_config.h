// kernel_config.h -- constants shared by the host planner (plan.cpp) and the decode
// kernel (decode_kernel.cu).  Product side only; the oracle never sees this file.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LORA_HD __host__ __device__ __forceinline__
#else
#define LORA_HD inline
#endif

namespace lora {

// ---- SIMT decode kernel (N1) -------------------------------------------------------
constexpr int kConsumerWarps = 8;                 // math warps
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kThreads = kConsumerThreads + 32;  // + one producer (bulk-copy) warp
constexpr int kStages = 3;                        // smem ring depth
constexpr int kTokChunk = 4;                      // tokens per (group, chunk)
constexpr int kShrinkRows = 8;                    // A rows per shrink unit
constexpr int kSliceBytes = 4096;                 // bytes of one A-row k-slice / one x-row k-slice
constexpr int kStageBytes = kShrinkRows * kSliceBytes + kTokChunk * kSliceBytes;  // 48 KB
constexpr int kExpandBytes = 32768;               // B bytes per expand unit (r * ncols * esz)
constexpr int kRedBytes = kConsumerThreads * kTokChunk * 8 * 4;  // 32 KB cross-part reduction
constexpr int kMetaSmemWords = 6144;              // metadata copied to smem when it fits (24 KB)

// metadata blob layout (int32 words)
constexpr int kHdrWords = 8;     // n_gc, n_shrink, n_expand, n_pages, n_toks, ksplit, pad, pad
constexpr int kGcFields = 8;     // rank, page_off, tok_off, ntok, shrink_base, expand_base, voff, scale_bits
enum { GC_RANK = 0, GC_PAGE_OFF, GC_TOK_OFF, GC_NTOK, GC_SHRINK_BASE, GC_EXPAND_BASE, GC_VOFF, GC_SCALE };

LORA_HD int vec_elems(int esz) { return 16 / esz; }             // elements per 16-B vector
LORA_HD int k_slice(int esz) { return kSliceBytes / esz; }       // k elements per shrink slice
LORA_HD int ksplit_of(int H_in, int esz) { return (H_in + k_slice(esz) - 1) / k_slice(esz); }
LORA_HD int pow2floor(int v) { int p = 1; while (p * 2 <= v) p *= 2; return p; }
// expand unit width in columns for rank r: largest power of two with r*ncols*esz <= kExpandBytes,
// capped at kConsumerThreads vectors (one 16-B vector per thread and part)
LORA_HD int expand_ncols(int r, int esz) {
    int c = pow2floor(kExpandBytes / (r * esz));
    int cap = kConsumerThreads * vec_elems(esz);
    return c < cap ? c : cap;
}
LORA_HD int shrink_jblocks(int r) { return (r + kShrinkRows - 1) / kShrinkRows; }

}  // namespace lora
