// plan.h -- host-side batch planner: canonical metadata (M1-M6) and kernel work lists.
// Step a1 of SURVEY.md §8(a): from seg_indptr / adapter_ids and the pool's id -> pages
// table, build the batch metadata "that parallelizes the LoRA weight gathering"
// (§4.1).  Pure C++ (no CUDA), so host-only pools exercise it on CPU.
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/lora_delta.h"
#include "kernel_config.h"

namespace lora {

struct AdapterRec {
    int32_t id = -1;
    int rank = 0;
    float scale = 1.f;
    std::vector<int32_t> pages;   // page indices, rank order
    void* ready = nullptr;        // cudaEvent_t of the load (owned by the pool)
    bool ready_known = false;
};

using AdapterTable = std::unordered_map<int32_t, AdapterRec>;

struct PrefillSeg {          // one tensor-core segment (N2 work)
    int32_t tok0, len, group;
};

struct Plan {
    // ---- canonical metadata (bit-exact contract, checked against oracle/) ----
    int32_t T = 0, S = 0, G = 0, L_tc = 64;
    std::vector<int32_t> tok_seg, group_id, group_rank, group_ntok, group_page_off, group_tok_off;
    std::vector<int32_t> group_tokens, pages, seg_kind;
    std::vector<float> group_scale;
    int64_t n_seg = 0, max_rank = 0, nseg_x_maxrank = 0, sum_rank_seg = 0, sum_rank_groups = 0,
            sum_rank_tokens = 0;
    // ---- SIMT decode kernel work (N1) ----
    std::vector<int32_t> blob;           // see kernel_config.h for the layout
    int32_t n_gc = 0, n_shrink = 0, n_expand = 0;
    int32_t unit_tab = 0;                // blob word offset of the per-unit table
    int32_t unit_words = kUnitWords;     // words per unit record: kUnitWords, or 1 for large batches
    int32_t blob_esz = 2;                // element size the unit table was built for
    int64_t vbuf_floats = 0;             // k-slice partials [gc][ksplit][ntok][v_stride(r)]
    int64_t vred_floats = 0;             // compact k-reduced v [gc][ntok][v_stride(r)] (TP payload)
    int32_t n_jobs = 1;                          // pools fused by lora_apply_multi
    int32_t job_shrink_base[4] = {0, 0, 0, 0};   // first shrink / expand unit of each job
    int32_t job_expand_base[4] = {0, 0, 0, 0};

    // ---- tcgen05 prefill work (N2) ----
    std::vector<PrefillSeg> prefill;
    int32_t n_prefill_tiles = 0;     // 128-token tiles on the tensor-core path (canonical count)
    std::vector<int32_t> pf_blob;    // [n_pf_tiles][8] CTA records {tok0, nvalid, rank, page_off, scale_bits,
                                     // first_page|-1, first column tile, end column tile}, then pages
    int32_t n_pf_tiles = 0;          // prefill CTAs (tiles x pf_cs)
    int32_t pf_cs = 1;               // CTAs per token tile (a cluster: split-K shrink + column split)

    // back to the default state but keeping every vector's capacity (one plan per apply: the
    // host planner is on the per-call path, so it should not reallocate)
    void reset() {
        std::vector<int32_t>* iv[] = {&tok_seg, &group_id, &group_rank, &group_ntok, &group_page_off, &group_tok_off,
                                      &group_tokens, &pages, &seg_kind, &blob, &pf_blob};
        for (auto* v : iv) v->clear();
        group_scale.clear();
        prefill.clear();
        Plan d;   // scalar defaults (its vectors are empty: no allocation)
        T = d.T; S = d.S; G = d.G; L_tc = d.L_tc;
        n_seg = max_rank = nseg_x_maxrank = sum_rank_seg = sum_rank_groups = sum_rank_tokens = 0;
        n_gc = n_shrink = n_expand = 0;
        unit_tab = 0; unit_words = d.unit_words; blob_esz = d.blob_esz; vbuf_floats = 0; vred_floats = 0; n_jobs = 1;
        for (int i = 0; i < 4; ++i) job_shrink_base[i] = job_expand_base[i] = 0;
        n_prefill_tiles = n_pf_tiles = 0;
        pf_cs = 1;
    }
};

// Builds `plan`.  tc_enabled=false routes every token through the SIMT kernel.  pad_zero_page >= 0
// pads every group's decode work to the batch's max rank with that (all-zero) page (BGMV mode;
// the canonical metadata M1-M6 is unchanged).
// Returns LORA_OK or an error status with `err` naming the offending operand.
lora_status build_plan(Plan& plan, const int32_t* seg_indptr, const int32_t* adapter_ids, int S,
                       int H_in, int H_out, int esz, int L_tc, bool tc_enabled,
                       const AdapterTable& table, std::string& err, int pad_zero_page = -1, int pf_sms = 0,
                       int expand_budget = 0);   // bytes per expand CTA, 0: single-pool rule (plan.cpp)

// ---- kernel launch descriptors (pool.cpp -> *_kernel.cu) ----
struct DecodeLaunch {
    const void* x;
    void* y;
    const void* poolA;
    const void* poolB;
    float* vbuf;
    int32_t* meta_dev;     // device scratch for metadata too large for kernel parameters
    unsigned long long* trace;   // optional per-unit timestamps (lora_debug_set_trace), or null
    int H_in, H_out, esz, num_sms;
    int phases = 3;              // bit 0: shrink kernel, bit 1: expand kernel
    float* vred = nullptr;       // phases 1: also reduce the partials over k-slices into this compact v;
                                 // phases 2: the expand reads this compact (k-reduced) v instead of vbuf
    int64_t x_ld = 0, y_ld = 0;  // row strides (elements) of x / y of job 0; 0 = H_in / H_out
    int* gc_cnt = nullptr;       // phases 1 with vred: the pool's zeroed per-gc arrival counters
    struct More {                // jobs 1.. of a fused multi-pool apply (job 0 = the fields above)
        const void* x;
        void* y;
        const void* poolA;
        const void* poolB;
        int H_in, H_out;
    } more[3];
    int n_jobs = 1;
};
struct PrefillLaunch {
    const void* x;
    void* y;
    const void* tm_a;      // 128-B CUtensorMap of the A pages (gather4 box {64, 1})
    const void* tm_b;      // 128-B CUtensorMap of the B pages
    const void* box_maps;  // device: the pool's 2D box maps (make_box_tmaps: A boxes {64, 8<<k}, then B)
    const int32_t* meta_dev;
    unsigned long long* trace;
    int T, H_in, H_out, zero_page, num_sms;
    float* pscratch = nullptr;   // split-K partials: [CTA][128 rows][128] fp32 (L2-resident exchange)
};

// Concatenates the SIMT work lists of plans[0..n) (one per fused pool = job index) into merged
// (only the kernel-work fields of merged are meaningful).
lora_status merge_plans(const Plan* const* plans, int n, Plan& merged, std::string& err);
}  // namespace lora

// implemented in the .cu files (declared here so host code needs no CUDA headers)
typedef struct CUstream_st* lora_cuda_stream;
namespace lora {
int launch_decode(const Plan& pl, const DecodeLaunch& L, lora_cuda_stream st, int* launches);
// zero-copy cold-start copy of one adapter (load_kernel.cu): sA/sB device-visible pinned host rows
int launch_load(char* dA, char* dB, const void* sA, const void* sB, int64_t ra, int64_t rb, int rank,
                const int32_t* pages, int num_sms, lora_cuda_stream st);
// writes the 2 * kBoxKinds CUtensorMaps (128 B each; A maps then B maps, box {64, 8 << k}) of a
// bf16 pool's page arrays to host_out; 0 on success
int make_box_tmaps(void* host_out, const void* dA, const void* dB, int n_rows, int H_in, int H_out);
int launch_prefill(const Plan& pl, const PrefillLaunch& L, lora_cuda_stream st, int* launches);

// NEXT f2: the delta fused into the base projection GEMM (fused_base_kernel.cu)
constexpr int kFusedBaseMaxWords = 7680;   // parameter blob: [tiles][8] records + page lists
struct FusedBaseLaunch {
    const void* x;      // [T][H_in] bf16
    const void* w;      // [H_in][H_out] bf16 (the base projection)
    void* y;            // [T][H_out] bf16, written
    const void* tm_a;   // the pool's gather4 maps
    const void* tm_b;
    int T, H_in, H_out, zero_page;
    const void* box_maps = nullptr;   // device: the pool's 2D box maps (contiguous adapters)
    const void* vtiles = nullptr;     // V tiles [n_vtiles * 128][v_cols] bf16 (written by the V items)
    int* vsync = nullptr;             // [2 + n_vtiles] ints, zero-initialised once, persistent (launch epochs)
    int n_vtiles = 0, v_cols = 0, n_vp = 0;   // n_vp: pairs with an adapter (ordered first)
    unsigned long long* trace = nullptr;      // lora_debug_set_trace buffer, or null
};
// words: [n_pairs][10] pair records {vtile, tok0_a, nvalid_a, tok0_b, nvalid_b (0: no partner), rank,
// page_off, scale_bits, first_page (-1: fragmented), 0}, then page lists (fused_base_kernel.cu)
int launch_fused_base(const FusedBaseLaunch& L, const int32_t* words, int n_words, int n_pairs, int num_sms,
                      lora_cuda_stream st);
bool prefill_supported(int H_in, int H_out, int esz);
int make_tmap_bf16(void* tm_out, const void* base, int64_t rows, int64_t cols, int box_rows);
constexpr int kPfMaxRank = 256;        // tensor-core prefill path handles ranks up to this (= LORA_MAX_RANK)
constexpr int kFusedMaxRank = 128;     // the fused base GEMM (f2): rank rows ride in one 128-row K chunk
constexpr int kPfMaxBlobWords = 7680;

}  // namespace lora
