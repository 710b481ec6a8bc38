// fused_base_kernel.cu -- SURVEY §8(f) NEXT row 2: the LoRA delta fused into the base projection
// GEMM (§4.1: "incorporate the operators of GPU LoRA computation into the base
// LLM inference process"; Eq. 1: y = x·W + x·A·B, with the per-adapter scale s).
//
// One launch: y = [x | V] · [W ; B_g] -- ONE GEMM whose K loop runs over H_in (x·W) and then over
// the adapter's rank (V·B_g): the expand is K-steps of the base MMA into the same TMEM accumulator, y
// is written once (never read), one bf16 rounding.  V = bf16(s_g · x·A_g) is computed inside the
// GEMM: each adapter pair's first column tile (a "V item", scheduled first) also issues the shrink
// MMAs D1 = x·A_g^T (N = rank) on its SMEM-resident x chunks into the idle second accumulator; its
// epilogue writes V to SMEM (its own rank K-steps) and to the pair's V tiles in global memory, where
// the pair's other column tiles find it behind a per-tile flag holding the launch's epoch (a device
// counter advanced by the last CTA of each launch: flags are never reset, graph replays stay valid).
// The GEMM is the sm_100 shape (DESIGN.md §6 F2): persistent CTA pairs (cluster of 2, tcgen05
// cta_group::2), 256 x 256 output tiles (each CTA: 128 token rows of the tile, half of the B
// columns in SMEM; the MMA reads both halves), a TMA ring of 32 KB stages per CTA (x or V chunk
// 128 x 64 K-major + W or B chunk 64 x 128 MN-major, SW128) plus a small ring of the adapter's A
// rows for V items, TMEM double-buffered accumulators (2 x 256 columns) so one tile's epilogue
// overlaps the next tile's mainloop.  Roles: warp 0 TMA producer (both CTAs: each loads its rows and
// its B half, signalling the leader's full barrier), warp 1 MMA issuer (leader CTA, one elected
// lane), warps 2-5 epilogue (TMEM -> bf16 -> SMEM -> coalesced stores, rows of the tile's segment
// only).  A pair's two 128-token tiles belong to one segment (one adapter: the K extension is
// uniform); an odd last tile runs with an empty partner.  A contiguous adapter's rank rows load as
// 2D boxes, the rest by tile::gather4 (zero page past the rank).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstring>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

constexpr int kFgThreads = 192;        // warp 0: TMA producer, warp 1: MMA issuer, warps 2-5: epilogue
#ifndef FG_STAGES
#define FG_STAGES 5
#endif
#ifndef FG_ASTAGES
#define FG_ASTAGES 4
#endif
constexpr int kFgStages = FG_STAGES;
constexpr int kFgAStages = FG_ASTAGES;   // V items: A-row ring depth
constexpr int kFgStageBytes = 32768;   // per CTA: A chunk (x or V) 16 KB + B chunk (W or B_g) 16 KB
constexpr int kFgAStageBytes = 8192;   // V items: this CTA's half of the adapter's A rows (<= 64 x 128 B)
constexpr int kFgEpiBytes = 4 * 2 * 2048;   // per epilogue warp: two 32-row x 64-B staging slots
constexpr int kFgSmem = 1024 + kFgStages * kFgStageBytes + kFgAStages * kFgAStageBytes + kFgEpiBytes + 256;
static_assert(kFgSmem <= 232448, "opt-in shared memory");
constexpr int kFgPairWords = 10;
#ifndef FG_B_KMAJOR
#define FG_B_KMAJOR 0   // experiment builds: 1 = W given as W^T [H_out][H_in] (nn.Linear layout), K-major B
#endif

struct FgArgs {
    CUtensorMap tm_x;   // x [T][H_in], box {64, 128}, SW128
    CUtensorMap tm_w;   // W [H_in][H_out], box {64, 64}, SW128 (MN-major atoms)
    CUtensorMap tm_v;   // V tiles [n_vtiles * 128][Rv], box {64, 128}, SW128
    CUtensorMap tm_b;   // B pages [n_pages+1][H_out], box {64, 1} (gather4)
    CUtensorMap tm_a;   // A pages [n_pages+1][H_in], box {64, 1} (gather4): the V items' shrink
    char* y;
    const char* box_maps;   // the pool's page arrays as 2D boxes {64, 8 << k}: A maps k, then B maps kBoxKinds + k
    char* vtiles;       // V tiles [n_vtiles * 128][v_cols] bf16, written by the V items
    int* vsync;         // [0] epoch of the last completed launch, [1] CTAs done, [2 + t] V tile t's epoch
    unsigned long long* trace;   // optional (lora_debug_set_trace): [cluster][64 items][4] globaltimer stamps
    int H_in, H_out, zero_page, n_items, n_ctiles, n_clusters, n_vp, n_ctas, v_cols;
};

struct FgBlob {
    int32_t w[kFusedBaseMaxWords];   // [n_pairs][8] pair records, then page lists
};

namespace {
__device__ __forceinline__ uint32_t fg_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void fg_bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fg_arrive_tx(uint32_t bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
// arrive on a barrier given by its shared::cluster address (this CTA's or the peer's)
__device__ __forceinline__ void fg_arrive_cluster(uint32_t cbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}
__device__ __forceinline__ void fg_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_FGW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_FGW;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t fg_mapa(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ uint32_t fg_cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void fg_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fg_prefetch_2d(const CUtensorMap* tm, int c0, int c1) {   // TMA box -> L2 only
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tm), "r"(c0), "r"(c1) : "memory");
}
// 2-CTA TMA: lands in this CTA's smem, completes on the LEADER's barrier (cluster address)
__device__ __forceinline__ void fg_tma_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t cbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(tm), "r"(c0), "r"(c1), "r"(cbar)
        : "memory");
}
__device__ __forceinline__ void fg_gather4(uint32_t dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                           uint32_t cbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(cbar)
        : "memory");
}
// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1 (sm_100)
__device__ __forceinline__ uint64_t fg_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D fp32, A/B bf16, A K-major, B MN-major (1) or K-major (0), M = 256 (CTA pair), N = 256
constexpr uint32_t fg_idesc(uint32_t b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn << 16) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
}
// executed by the whole (converged) warp; one elected lane issues (warp-uniform operands stay in
// uniform registers: no per-lane waterfall around the instruction)
__device__ __forceinline__ void fg_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// commit the leader's MMAs so far: arrive on the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void fg_commit2(uint32_t bar) {   // whole warp; one elected lane commits
    asm volatile(
        "{\n\t.reg .b16 m;\n\t.reg .pred e;\n\tmov.b16 m, 3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ unsigned long long fg_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void fg_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fg_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fg_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
}  // namespace

// work item w -> (token pair p, column tile ct, computes V?).  Pairs with an adapter come first
// (p < n_vp); items 0 .. n_vp-1 are their column tile 0 and also run the shrink (the "V items"),
// scheduled first so the pairs' other column tiles rarely wait for V; then the rest, pair-major.
struct FgItem {
    int p, ct;
    bool vit;
};
__device__ __forceinline__ FgItem fg_item(int w, int n_vp, int C) {
    if (w < n_vp) return {w, 0, true};
    int j = w - n_vp;
    if (C > 1 && j < n_vp * (C - 1)) return {j / (C - 1), 1 + j % (C - 1), false};
    j -= n_vp * (C - 1);
    return {n_vp + j / C, j % C, false};
}
__device__ __forceinline__ int fg_ld_relaxed(const int* p) {   // no ordering: later loads/TMAs are not held back
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fg_st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fg_fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Rank rows [row0, row0 + nrows) of an adapter of rank r, 64 columns from `col`, into dst (row i at
// dst + 128 i: SW128 atoms of 8 rows, the layout of both the K-major A rows and the MN-major B rows).
// A contiguous adapter's rows below r (rounded down to 8) go as 2D boxes of 64/32/16/8 rows -- one TMA
// request instead of one per 4 rows (the request rate bounds gather4-only loads); the rest, and
// every row of a fragmented adapter, by tile::gather4 with the pool's zero page past r (never a
// neighbouring tenant's page).  Called by the whole warp; 128·nrows bytes complete on cbar.
__device__ __forceinline__ void fg_load_rows(uint32_t dst, const char* box_maps, int map_base, const CUtensorMap* g4map,
                                             int col, int first_page, const int32_t* pages, int row0, int nrows, int r,
                                             int zero_page, uint32_t cbar, int lane) {
    const int valid = min(max(r - row0, 0), nrows);
    const int rb = (first_page >= 0 && box_maps != nullptr) ? (valid & ~7) : 0;
    if (lane == 0) {
        int row = 0;
        for (int k = 3; k >= 0; --k) {   // boxes of 64 / 32 / 16 / 8 rows
            const int R = 8 << k;
            while (rb - row >= R) {
                fg_tma_2d(dst + (uint32_t)row * 128u, reinterpret_cast<const CUtensorMap*>(box_maps + (map_base + k) * 128),
                          col, first_page + row0 + row, cbar);
                row += R;
            }
        }
    }
    const int ng = (nrows - rb + 3) >> 2;
    for (int gi = lane; gi < ng; gi += 32) {
        int pg[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = row0 + rb + 4 * gi + i;
            pg[i] = j < r ? pages[j] : zero_page;
        }
        fg_gather4(dst + (uint32_t)(rb + 4 * gi) * 128u, g4map, col, pg[0], pg[1], pg[2], pg[3], cbar);
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFgThreads, 1)
    lora_fused_gemm_kernel(const __grid_constant__ FgArgs a, const __grid_constant__ FgBlob blob) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = fg_smem(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;   // SW128 atoms need 1 KB alignment
    uint8_t* gbase = smem_raw + (base - raw);
    const uint32_t ring = base;
    const uint32_t aring = base + kFgStages * kFgStageBytes;       // V items: adapter A rows, kFgAStages x 8 KB
    const uint32_t epi = aring + kFgAStages * kFgAStageBytes;
    const uint32_t bars = epi + kFgEpiBytes;
    auto full = [&](int s) { return bars + 8u * s; };                       // leader's is the live one
    auto empty = [&](int s) { return bars + 8u * (kFgStages + s); };         // both CTAs (MMA commit multicast)
    auto tfull = [&](int b) { return bars + 8u * (2 * kFgStages + b); };     // both CTAs
    auto tempty = [&](int b) { return bars + 8u * (2 * kFgStages + 2 + b); };   // leader: both epilogues arrive
    auto afull = [&](int s) { return bars + 8u * (2 * kFgStages + 4 + s); };    // leader
    auto aempty = [&](int s) { return bars + 8u * (2 * kFgStages + 4 + kFgAStages + s); };   // both CTAs
    constexpr int kB0 = 2 * kFgStages + 4 + 2 * kFgAStages;
    const uint32_t d1full = bars + 8u * kB0;                  // both CTAs
    const uint32_t vsm_full = bars + 8u * (kB0 + 1);          // leader: both CTAs' V in SMEM
    const uint32_t vsm_free = bars + 8u * (kB0 + 2);          // both CTAs: V-item rank MMAs done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars + 8u * (kB0 + 3) - base));
    static_assert(8 * (kB0 + 3) + 4 <= 256, "barrier block");
    // a V item's V (128 rows x rank, bf16 K-major SW128, two 64-column atoms) lives in the A-row ring
    // and the epilogue staging (contiguous 32 KB; both idle then) for its own rank K steps
    const uint32_t vsm = aring;
    static_assert(kFgAStages * kFgAStageBytes + kFgEpiBytes >= 32768, "V atoms in the A-row ring (+ epilogue staging)");

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t crank = fg_cta_rank();
    const bool leader = crank == 0;
    const int cluster = blockIdx.x >> 1;
    const int nkc = a.H_in / 64;

    if (tid == 0) {
        for (int s = 0; s < kFgStages; ++s) {
            fg_bar_init(full(s), 1);
            fg_bar_init(empty(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            fg_bar_init(tfull(b), 1);
            fg_bar_init(tempty(b), 2);
        }
        for (int s = 0; s < kFgAStages; ++s) {
            fg_bar_init(afull(s), 1);
            fg_bar_init(aempty(s), 1);
        }
        fg_bar_init(d1full, 1);
        fg_bar_init(vsm_full, 2);
        fg_bar_init(vsm_free, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // both CTAs: two 256-column fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(fg_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fg_fence_before();
    fg_cluster_sync();   // the peer's barriers are initialised before any remote arrive / TMA complete_tx
    __syncthreads();     // (also orders the TMEM address write before every reader, as racecheck models it)
    fg_fence_after();
    const uint32_t tmem = *tmem_slot;
    // x, W, y and the V-sync words may belong to preceding kernels in the stream
    if (tid == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // this launch's epoch: V-tile flags equal to it were published by this launch (never reset)
    const int epoch = a.vsync ? *reinterpret_cast<volatile const int*>(a.vsync) + 1 : 0;   // (no adapter: none)
    int* vflag = a.vsync + 2;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        const uint32_t lfull0 = fg_mapa(full(0), 0);     // the leader's full barrier 0 (cluster address)
        const uint32_t lafull0 = fg_mapa(afull(0), 0);
        int stage = 0, astage = 0, nvi = 0;
        uint32_t phase = 0, aphase = 0;
        for (int w = cluster; w < a.n_items; w += a.n_clusters) {
            const FgItem itm = fg_item(w, a.n_vp, a.n_ctiles);
            const int32_t* rec = blob.w + itm.p * kFgPairWords;
            const bool solo = rec[4] == 0;
            const int tok0 = crank == 0 || solo ? rec[1] : rec[3];
            const int vtile = rec[0] + (crank == 0 || solo ? 0 : 1);
            const int r = rec[5], poff = rec[6];
            const int rp = (r + 15) & ~15;
            const int nch = nkc + (rp + 63) / 64;
            const int nb0 = itm.ct * 256 + (int)crank * 128;   // this CTA's half of the B columns
            // an item that is not its pair's V item reads V from the V tiles: the flag load is issued
            // now and checked at the rank chunks (another CTA pair stores V, flag = this launch's epoch)
            // lane 1 owns the V-tile flag, its fences and the V-tile TMA loads: lane 0 has TMA loads in
            // flight, which a proxy fence on lane 0 would wait for
            int vf = 0;
            if (!itm.vit && r > 0 && lane == 1) vf = fg_ld_relaxed(vflag + vtile);
            // the rank chunks' operands are read ~20 us from now: into L2 at the item's start (V tile rows
            // -- stale lines are harmless, the V stores update L2 -- and a contiguous adapter's B rows)
            if (r > 0 && lane == 0) {
                if (!itm.vit)
                    for (int e = 0; e * 64 < rp; ++e) fg_prefetch_2d(&a.tm_v, e * 64, vtile * 128);
                if (rec[8] >= 0 && a.box_maps)
                    for (int h = 0; h < 2; ++h)
                        for (int row = 0; row < rp; row += 64)
                            fg_prefetch_2d(reinterpret_cast<const CUtensorMap*>(a.box_maps + (kBoxKinds + 3) * 128),
                                           nb0 + h * 64, rec[8] + row);
            }
            if (itm.vit && nvi++ > 0) fg_wait(vsm_free, (uint32_t)((nvi - 2) & 1));   // previous V item's V read
            for (int kc = 0; kc < nch; ++kc) {
                if (kc == nkc && !itm.vit && lane == 1) {
                    while (vf != epoch) {
                        __nanosleep(64);
                        vf = fg_ld_relaxed(vflag + vtile);
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");   // acquire: the flag's V stores
                    fg_fence_proxy_global();   // generic-proxy V stores -> the async-proxy TMA reads below
                }
                fg_wait(empty(stage), phase ^ 1u);
                const uint32_t sb = ring + (uint32_t)stage * kFgStageBytes;
                const uint32_t cbar = lfull0 + 8u * (uint32_t)stage;
                if (kc < nkc) {
                    if (lane == 0) {
                        if (leader) fg_arrive_tx(full(stage), 2u * kFgStageBytes);
                        fg_tma_2d(sb, &a.tm_x, kc * 64, tok0, cbar);
#if FG_B_KMAJOR
                        fg_tma_2d(sb + 16384, &a.tm_w, kc * 64, nb0, cbar);   // W^T [H_out][H_in]: box {64 K, 128 N}
#else
                        fg_tma_2d(sb + 16384, &a.tm_w, nb0, kc * 64, cbar);
                        fg_tma_2d(sb + 16384 + 8192, &a.tm_w, nb0 + 64, kc * 64, cbar);
#endif
                    }
                    if (itm.vit) {
                        // the shrink's B operand: this CTA's half of the adapter's A rank rows for this
                        // K chunk, rows [crank * rp/2, +rp/2), gather4 with the zero page past r
                        fg_wait(aempty(astage), aphase ^ 1u);
                        if (leader && lane == 0) fg_arrive_tx(afull(astage), (uint32_t)(rp * 128));
                        __syncwarp();
                        fg_load_rows(aring + (uint32_t)astage * kFgAStageBytes, a.box_maps, 0, &a.tm_a, kc * 64, rec[8],
                                     blob.w + poff, (int)crank * (rp / 2), rp / 2, r, a.zero_page,
                                     lafull0 + 8u * (uint32_t)astage, lane);
                        if (++astage == kFgAStages) { astage = 0; aphase ^= 1u; }
                    }
                } else {
                    const int e = kc - nkc;
                    // only the rank rows the MMA reads: [64e, min(64e + 64, rp)) (rows r..rp-1 from the
                    // zero page); a V item's V is already in SMEM, so only the B rows
                    const int rows = min(64, rp - 64 * e);
                    if (lane == 0 && leader)
                        fg_arrive_tx(full(stage), (uint32_t)(2 * (itm.vit ? 0 : 16384) + 2 * 2 * rows * 128));
                    if (lane == 1 && !itm.vit) fg_tma_2d(sb, &a.tm_v, e * 64, vtile * 128, cbar);
                    __syncwarp();
                    // the B rank rows [64e, 64e + 64) of each 64-column half of this CTA's B columns
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        fg_load_rows(sb + 16384 + (uint32_t)h * 8192u, a.box_maps, kBoxKinds, &a.tm_b, nb0 + h * 64, rec[8],
                                     blob.w + poff, e * 64, rows, r, a.zero_page, cbar, lane);
                }
                __syncwarp();
                if (++stage == kFgStages) { stage = 0; phase ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA, one elected lane) =====================
        // Descriptors are built once and advanced by adding to their start-address field (addr >> 4,
        // low 14 bits): +2 per 32-B K step of the K-major A / K-major B atoms, +128 per 2 KB K step of
        // the MN-major B atoms, +2048 per 32 KB ring stage.  The x·W chunks issue their 4 K steps
        // unrolled; only the adapter-rank chunks have a variable step count.  A V item also runs the
        // shrink D1 = x·A_g^T (N = rank) on the same x chunks into the other accumulator buffer.
        if (leader) {
            const uint64_t a0 = fg_desc(ring, 16, 1024);
            const uint64_t b0 = FG_B_KMAJOR ? fg_desc(ring + 16384, 16, 1024) : fg_desc(ring + 16384, 8192, 1024);
            const uint64_t be0 = fg_desc(ring + 16384, 8192, 1024);   // adapter B rows: MN-major
            const uint64_t ar0 = fg_desc(aring, 16, 1024);             // adapter A rows: K-major
            const uint64_t v0 = fg_desc(vsm, 16, 1024);                // a V item's V: K-major
            int nvm = 0;
            constexpr uint64_t kBStep = FG_B_KMAJOR ? 2 : 128;
            constexpr uint32_t kIdW = fg_idesc(FG_B_KMAJOR ? 0u : 1u), kIdB = fg_idesc(1u);
            int stage = 0, astage = 0, it = 0;
            uint32_t phase = 0, aphase = 0;
            uint32_t tph[2] = {1u, 1u};   // tempty wait parity per buffer (flips per use)
            for (int w = cluster; w < a.n_items; w += a.n_clusters, ++it) {
                const FgItem itm = fg_item(w, a.n_vp, a.n_ctiles);
                const int r = blob.w[itm.p * kFgPairWords + 5];
                const int rp = (r + 15) & ~15;
                const int nch = nkc + (rp + 63) / 64;
                const int b = it & 1;
                fg_wait(tempty(b), tph[b]);   // both epilogues drained this accumulator
                tph[b] ^= 1u;
                if (itm.vit) {                // D1 goes into the other buffer: drained as well
                    fg_wait(tempty(b ^ 1), tph[b ^ 1]);
                    tph[b ^ 1] ^= 1u;
                }
                fg_fence_after();
                unsigned long long* trc = a.trace && it < 64 ? a.trace + ((size_t)cluster * 64 + it) * 4 : nullptr;
                if (trc && lane == 0) trc[0] = fg_gtime();
                const uint32_t dacc = tmem + (uint32_t)b * 256u;
                const uint32_t d1 = tmem + (uint32_t)(b ^ 1) * 256u;
                const uint32_t id1 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(rp >> 3) << 17) | ((256u >> 4) << 24);
                for (int kc = 0; kc < nch; ++kc) {
                    fg_wait(full(stage), phase);
                    fg_fence_after();
                    const uint64_t so = (uint64_t)stage * (kFgStageBytes >> 4);
                    const uint64_t ad = a0 + so;
                    if (kc < nkc) {
                        const uint64_t bd = b0 + so;
                        fg_mma2(dacc, ad, bd, kIdW, kc != 0);
                        fg_mma2(dacc, ad + 2, bd + kBStep, kIdW, 1u);
                        fg_mma2(dacc, ad + 4, bd + 2 * kBStep, kIdW, 1u);
                        fg_mma2(dacc, ad + 6, bd + 3 * kBStep, kIdW, 1u);
                        if (itm.vit) {
                            fg_wait(afull(astage), aphase);
                            fg_fence_after();
                            const uint64_t sd = ar0 + (uint64_t)astage * (kFgAStageBytes >> 4);
                            fg_mma2(d1, ad, sd, id1, kc != 0);
                            fg_mma2(d1, ad + 2, sd + 2, id1, 1u);
                            fg_mma2(d1, ad + 4, sd + 4, id1, 1u);
                            fg_mma2(d1, ad + 6, sd + 6, id1, 1u);
                            fg_commit2(aempty(astage));
                            if (kc == nkc - 1) fg_commit2(d1full);
                            if (++astage == kFgAStages) { astage = 0; aphase ^= 1u; }
                        }
                    } else {
                        const int e = kc - nkc;
                        const uint64_t bd = be0 + so;
                        uint64_t av = ad;
                        if (itm.vit) {   // V from SMEM, written by both CTAs' epilogues
                            if (e == 0) {
                                fg_wait(vsm_full, (uint32_t)(nvm & 1));
                                ++nvm;
                                fg_fence_after();
                            }
                            av = v0 + (uint64_t)e * (16384 >> 4);
                        }
                        const int ks = min(4, (rp - e * 64) / 16);
                        for (int kk = 0; kk < ks; ++kk) fg_mma2(dacc, av + 2 * kk, bd + 128 * kk, kIdB, 1u);
                        if (itm.vit && kc == nch - 1) fg_commit2(vsm_free);
                    }
                    fg_commit2(empty(stage));
                    if (kc == nch - 1) fg_commit2(tfull(b));
                    if (trc && lane == 0 && kc == nkc - 1) trc[1] = fg_gtime();
                    __syncwarp();
                    if (++stage == kFgStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else {
        // ===================== epilogue: warps 2..5 -> TMEM lanes 32*(warp%4) .. +32 =====================
        const int sub = warp & 3;
        const int row = sub * 32 + lane;   // token row of this CTA's 128
        const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
        const uint32_t ltempty0 = fg_mapa(tempty(0), 0);
        const uint32_t lvsmfull = fg_mapa(vsm_full, 0);
        uint8_t* stg0 = gbase + (epi - base) + sub * 4096;
        int it = 0, nd = 0;
        for (int w = cluster; w < a.n_items; w += a.n_clusters, ++it) {
            const FgItem itm = fg_item(w, a.n_vp, a.n_ctiles);
            const int32_t* rec = blob.w + itm.p * kFgPairWords;
            const bool solo = rec[4] == 0;
            const int tok0 = crank == 0 ? rec[1] : rec[3];
            const int nvalid = crank == 0 ? rec[2] : (solo ? 0 : rec[4]);
            const int b = it & 1;
            if (itm.vit) {
                // V = bf16(s · D1) of this CTA's 128 token rows -> its V tile (rows past the segment are
                // never read: their y rows are not stored); then D1's buffer is free again
                const int r = rec[5], rp = (r + 15) & ~15;
                const float scale = __int_as_float(rec[7]);
                const int vtile = rec[0] + (crank == 0 ? 0 : 1);
                fg_wait(d1full, (uint32_t)(nd & 1));
                ++nd;
                fg_fence_after();
                const bool vwriter = crank == 0 || !solo;
                uint8_t* gvsm = gbase + (vsm - base);
                {
                    // every CTA (a solo pair's second CTA too: its rows feed only unstored y rows) puts its
                    // V rows into SMEM for the rank K steps; writers also store them to their V tile
                    char* vrow = a.vtiles + ((size_t)vtile * 128 + row) * a.v_cols * 2;
                    for (int c0 = 0; c0 < rp; c0 += 32) {
                        float v[32];
                        fg_ld32(tmem + lane_addr + (uint32_t)(b ^ 1) * 256u + (uint32_t)c0, v);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint32_t o[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int j0 = c0 + q * 8 + 2 * e;
                                __nv_bfloat162 hb = __floats2bfloat162_rn(j0 < r ? v[q * 8 + 2 * e] * scale : 0.f,
                                                                          j0 + 1 < r ? v[q * 8 + 2 * e + 1] * scale : 0.f);
                                o[e] = *reinterpret_cast<uint32_t*>(&hb);
                            }
                            const int col = c0 + q * 8;
                            if (col < rp) {
                                const uint4 v4 = make_uint4(o[0], o[1], o[2], o[3]);
                                if (vwriter) *reinterpret_cast<uint4*>(vrow + col * 2) = v4;
                                // K-major SW128: atom col/64, row at (row/8)*1024 + (row%8)*128, chunk ^ row%8
                                const int kk = col >> 6, chunk = (col & 63) >> 3;
                                *reinterpret_cast<uint4*>(gvsm + kk * 16384 + (row >> 3) * 1024 + (row & 7) * 128 +
                                                          ((chunk ^ (row & 7)) << 4)) = v4;
                            }
                        }
                    }
                    if (vwriter) {
                        fg_fence_proxy_global();
                        __threadfence();
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // -> the tensor core's reads
                }
                fg_fence_before();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tid == 64) {
                    fg_arrive_cluster(ltempty0 + 8u * (uint32_t)(b ^ 1));   // D1's accumulator drained
                    fg_arrive_cluster(lvsmfull);                            // this CTA's V is in SMEM
                    if (vwriter) fg_st_release(a.vsync + 2 + vtile, epoch);  // for the pair's other column tiles
                }
            }
            fg_wait(tfull(b), (uint32_t)((it >> 1) & 1));
            fg_fence_after();
            unsigned long long* trc = a.trace && leader && it < 64 ? a.trace + ((size_t)cluster * 64 + it) * 4 : nullptr;
            if (trc && tid == 64) trc[2] = fg_gtime() | ((unsigned long long)(itm.vit ? 1 : 0) << 63);
            const int n0 = itm.ct * 256;
#pragma unroll 1
            for (int c0 = 0; c0 < 256; c0 += 32) {
                float d[32];
                fg_ld32(tmem + lane_addr + (uint32_t)b * 256u + (uint32_t)c0, d);
                uint8_t* stg = stg0 + ((c0 >> 5) & 1) * 2048;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        __nv_bfloat162 hb = __floats2bfloat162_rn(d[q * 8 + 2 * e], d[q * 8 + 2 * e + 1]);
                        o[e] = *reinterpret_cast<uint32_t*>(&hb);
                    }
                    *reinterpret_cast<uint4*>(stg + lane * 64 + ((q + lane) & 3) * 16) = make_uint4(o[0], o[1], o[2], o[3]);
                }
                __syncwarp();
                // 32 rows x 64 B leave as 8 rows x 64 contiguous bytes per store instruction
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int idx = i * 32 + lane, rr = idx >> 2, qq = idx & 3;
                    const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * 64 + ((qq + rr) & 3) * 16);
                    if (sub * 32 + rr < nvalid)
                        *reinterpret_cast<uint4*>(a.y + ((size_t)(tok0 + sub * 32 + rr) * a.H_out + n0 + c0 + qq * 8) * 2) = v;
                }
            }
            // this CTA's 128 TMEM lanes of accumulator b are drained -> one arrival on the leader's barrier
            fg_fence_before();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tid == 64) fg_arrive_cluster(ltempty0 + 8u * (uint32_t)b);
            if (trc && tid == 64) trc[3] = fg_gtime();
        }
    }
    fg_fence_before();
    __syncthreads();
    fg_cluster_sync();   // the peer's MMAs (leader) are done with this CTA's smem and TMEM
    if (warp == 1) {
        fg_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
    // the last CTA out publishes this launch's epoch (the next launch's flags must differ)
    if (tid == 0 && a.vsync) {
        __threadfence();
        const int done = atomicAdd(a.vsync + 1, 1);
        if (done == a.n_ctas - 1) {
            a.vsync[1] = 0;
            __threadfence();
            a.vsync[0] = epoch;
        }
    }
}

int make_tmap_bf16(void* tm_out, const void* base, int64_t rows, int64_t cols, int box_rows);   // prefill_kernel.cu

int launch_fused_base(const FusedBaseLaunch& L, const int32_t* words, int n_words, int n_pairs, int num_sms,
                      lora_cuda_stream st) {
    if (n_words > kFusedBaseMaxWords || n_pairs <= 0 || L.H_out % 256 || L.H_in % 64) return (int)cudaErrorInvalidValue;
    if (L.n_vp > 0 && (!L.vtiles || !L.vsync)) return (int)cudaErrorInvalidValue;
    FgArgs a;
    std::memset(&a, 0, sizeof(a));
    int e = make_tmap_bf16(&a.tm_x, L.x, L.T, L.H_in, 128);
#if FG_B_KMAJOR
    if (!e) e = make_tmap_bf16(&a.tm_w, L.w, L.H_out, L.H_in, 128);   // experiment: W^T [H_out][H_in]
#else
    if (!e) e = make_tmap_bf16(&a.tm_w, L.w, L.H_in, L.H_out, 64);
#endif
    if (!e && L.n_vp > 0) e = make_tmap_bf16(&a.tm_v, L.vtiles, (int64_t)L.n_vtiles * 128, L.v_cols, 128);
    else if (!e) e = make_tmap_bf16(&a.tm_v, L.x, L.T, L.H_in, 128);   // (no adapter: never loaded)
    if (e) return e;
    std::memcpy(&a.tm_b, L.tm_b, sizeof(CUtensorMap));
    std::memcpy(&a.tm_a, L.tm_a, sizeof(CUtensorMap));
    a.y = static_cast<char*>(L.y);
    a.vtiles = static_cast<char*>(const_cast<void*>(L.vtiles));
    a.vsync = L.vsync;
    a.v_cols = L.v_cols;
    a.box_maps = static_cast<const char*>(L.box_maps);
    a.trace = L.trace;
    a.H_in = L.H_in;
    a.H_out = L.H_out;
    a.zero_page = L.zero_page;
    a.n_ctiles = L.H_out / 256;
    a.n_items = n_pairs * a.n_ctiles;
    a.n_vp = L.n_vp;
    a.n_clusters = std::min(a.n_items, std::max(1, num_sms / 2));
    a.n_ctas = 2 * a.n_clusters;
    FgBlob blob;   // the kernel-parameter blob (copied into the launch)
    std::memcpy(blob.w, words, (size_t)n_words * 4);
    // cudaFuncSetAttribute is per device: one bit per device
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return (int)cudaErrorInvalidDevice;
    const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;
    if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
        cudaError_t ce = cudaFuncSetAttribute(lora_fused_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFgSmem);
        if (ce != cudaSuccess) return (int)ce;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_ctas);
    cfg.blockDim = dim3(kFgThreads);
    cfg.dynamicSmemBytes = kFgSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, lora_fused_gemm_kernel, a, blob);
}

}  // namespace lora
