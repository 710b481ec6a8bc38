// kernel_config.h -- constants shared by the host planner (plan.cpp) and the decode
// kernels (decode_kernel.cu).  Product side only; the oracle never sees this file.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LORA_HD __host__ __device__ __forceinline__
#else
#define LORA_HD inline
#endif

namespace lora {

// ---- decode kernels (N1) ------------------------------------------------------------
constexpr int kConsumerWarps = 8;                 // warps per CTA
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kTokChunk = 4;                      // fp32 SIMT kernels: tokens per (group, chunk)
constexpr int kTokChunkMma = 8;                   // bf16 tensor-core kernels: tokens per chunk (MMA N = 8)
constexpr int kMaxTokChunk = 8;
constexpr int kShrinkRows = 8;                    // fp32: A rows per shrink unit
constexpr int kShrinkRowsMma = 16;                // bf16: A rows per shrink unit (MMA M = 16)
#ifndef LORA_KSLICE
#define LORA_KSLICE 1024                          // experiment builds: LORA_BUILD_DEFS=-DLORA_KSLICE=2048
#endif
constexpr int kKSlice = LORA_KSLICE;              // k elements per shrink unit (both element types)
constexpr int kSliceBytes = kKSlice * 4;          // fp32 smem row slice
constexpr int kExpandBytes = 32768;               // fp32 SIMT expand: B bytes per unit (r * ncols * esz)
constexpr int kMaxNcols = 1024;                   // fp32 SIMT expand: columns per unit
#ifndef LORA_EXPAND_MAXC
#define LORA_EXPAND_MAXC 2048
#endif
constexpr int kMaxNcolsMma = LORA_EXPAND_MAXC;    // bf16 expand: columns per unit
// bf16 expand CTA budget: its whole SMEM (v tiles, B rows, staged y rows, fp32 D^T, pages) fits
// 4 CTAs per SM (228 KB per SM, 1 KB reserved per CTA), so an expand grid of <= 4 x 148 units --
// q/k/v of a c2 decode batch in one lora_apply_multi -- is resident in ONE wave
#ifndef LORA_EXPAND_BUDGET
#define LORA_EXPAND_BUDGET (56 * 1024)
#endif
constexpr int kExpandSmemBudget = LORA_EXPAND_BUDGET;
constexpr int kExpandSmemBudget3 = 75 * 1024;   // the largest bf16 expand CTA of which 3 share an SM

// metadata blob layout (int32 words)
constexpr int kHdrWords = 8;     // n_gc, n_shrink, n_expand, n_pages, n_toks, ksplit, unit_tab, pad
// blob = header | gc records [n_gc][kGcFields] | pages | tokens | unit table [n_shrink + n_expand]
// (unit record = kUnitWords words, see plan.cpp append_unit_table)
constexpr int kUnitWords = 3;
constexpr int kMaxParamBlobWords = 7936;   // largest metadata blob passed as kernel parameters
// A page reference is either a blob word offset of an explicit page list (>= 0) or, for a run of
// consecutive pages, ~first_page (< 0): page j = first_page + j.  Contiguous adapters (the
// allocator's lowest-free-first order makes them the common case) then cost no blob words.
LORA_HD int page_ref_add(int ref, int k) { return ref >= 0 ? ref + k : ~((~ref) + k); }
// unit word 2: rank | ntok << 9 | token offset << 13
LORA_HD int unit_rank(uint32_t w) { return (int)(w & 0x1ffu); }
LORA_HD int unit_ntok(uint32_t w) { return (int)((w >> 9) & 0xfu); }
LORA_HD int unit_tok_off(uint32_t w) { return (int)(w >> 13); }
constexpr int kGcFields = 11;    // rank, page_off, tok_off, ntok, shrink_base, expand_base, voff, scale_bits, job,
                                 // vred (offset of the gc's k-reduced v [ntok][v_stride(r)] in the compact v),
                                 // ncols (expand unit width of the gc: expand_cols_gc)
enum { GC_RANK = 0, GC_PAGE_OFF, GC_TOK_OFF, GC_NTOK, GC_SHRINK_BASE, GC_EXPAND_BASE, GC_VOFF, GC_SCALE, GC_JOB, GC_VRED,
       GC_NCOLS };
constexpr int kMaxJobs = 4;      // pools fused into one launch pair by lora_apply_multi (e.g. q, k, v)

constexpr int kBoxKinds = 5;                      // 2D TMA boxes {64 columns, 8 << k page rows}, k < 5

LORA_HD int vec_elems(int esz) { return 16 / esz; }             // elements per 16-B vector
LORA_HD int tok_chunk(int esz) { return esz == 2 ? kTokChunkMma : kTokChunk; }
LORA_HD int shrink_rows(int esz) { return esz == 2 ? kShrinkRowsMma : kShrinkRows; }
LORA_HD int ksplit_of(int H_in, int /*esz*/) { return (H_in + kKSlice - 1) / kKSlice; }
LORA_HD int pow2floor(int v) { int p = 1; while (p * 2 <= v) p *= 2; return p; }
// expand unit width in columns for rank r: largest power of two with r*ncols*esz <= kExpandBytes,
// capped at kMaxNcols
LORA_HD int expand_ncols(int r, int esz) {
    int c = pow2floor(kExpandBytes / (r * esz));
    return c < kMaxNcols ? c : kMaxNcols;
}
// bf16 expand unit SMEM (decode_kernel.cu expand_mma_body layout): [0,320) barriers, unit record,
// 64 zero bytes | v as bf16 (hi, lo) pairs [token groups of 4][8][rp + 8] | B rows [r][nc + 8] |
// y rows [ntok][nc + 8] | fp32 D^T [ntok][nc + 4] | pages [r]
LORA_HD int expand_mma_boff(int r, int ntok) {
    return (320 + ((ntok + 3) >> 2) * 8 * (((r + 15) & ~15) + 8) * 2 + 127) & ~127;
}
LORA_HD int expand_mma_smem(int r, int nc, int ntok) {
    const int pitch = nc * 2 + 16;
    return expand_mma_boff(r, ntok) + r * pitch + ntok * pitch + ntok * (nc + 4) * 4 + r * 4;
}
// expand unit width of a gc (columns, the last unit of a gc may be narrower).  fp32: the power-of-two
// rule above.  bf16: as few units as fit kExpandSmemBudget each -- widths are multiples of 16 (MMA
// tiles; an odd number of 16-B vectors in the SMEM row pitch keeps ldmatrix conflict-free), not
// powers of two, so a gc's B bytes split into near-equal units (budget 0: the power-of-two rule)
LORA_HD int expand_cols_gc(int r, int ntok, int H_out, int esz, int budget) {
    if (esz != 2 || budget <= 0) return expand_ncols(r, esz);   // budget 0: round 1's power-of-two units
    for (int nu = (H_out + kMaxNcolsMma - 1) / kMaxNcolsMma;; ++nu) {
        const int nc = ((H_out + nu - 1) / nu + 15) & ~15;
        if (nc <= 16 || expand_mma_smem(r, nc, ntok) <= budget) return nc;
    }
}
// row stride of a gc's rank-r intermediate in the v scratch: r rounded up to 4 floats, so every
// [k-slice][token] row starts 16-B aligned (float4 loads) -- layout [ksplit][ntok][v_stride(r)]
LORA_HD int v_stride(int r) { return (r + 3) & ~3; }
LORA_HD int shrink_jblocks(int r, int esz) { return (r + shrink_rows(esz) - 1) / shrink_rows(esz); }

}  // namespace lora
