// prefill_kernel.cu -- N2: the LoRA delta of long prefill segments on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
// For a segment of tokens [t0, t0+len) on adapter g (rank r <= 256), per 128-token tile:
//     V[t][j]  = s_g · Σ_k X[t][k] · A_g[k][j]      shrink  D1[128 x r16] in TMEM  (Eq. 1)
//     Y[t][n] += Σ_j V[t][j] · B_g[j][n]            expand  D2[128 x 128] in TMEM, per 128-column tile
//
// * X tiles arrive by TMA (2D tiled, SWIZZLE_128B); the adapter's rank rows are gathered from
//   the paged pool by TMA tile::gather4 (4 page rows per instruction) straight into the
//   canonical UMMA smem layouts: A rows K-major for the shrink, B rows MN-major for the
//   expand (no transposition anywhere).  Rank padding to a multiple of 16 uses the pool's
//   all-zero page, in SMEM only.
// * One elected thread issues tcgen05.mma (M=128, kind::f16, bf16 inputs, fp32 accumulate);
//   tcgen05.commit releases ring slots and signals the epilogue.
// * The epilogue (4 warps = the 128 TMEM lanes) reads D1, applies s_g and rounds v once to
//   bf16, written as the expand's A operand (K-major SW128; reading R4) -- then, per
//   expand tile, reads D2 and adds it to y with one rounding.  D2 is double-buffered in TMEM so
//   the epilogue of tile n overlaps the MMAs of tile n+1.
// The path is HBM-bound (x read once, y read+written once per tile; adapter rows mostly
// from L2), so tensor-pipe utilisation is reported next to the HBM roofline.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstring>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

// warp 0: TMA producer, warp 1: MMA issuer, warps 2-5 and 6-9: two epilogue groups (each the 128
// TMEM lanes) taking the expand tiles alternately, one per TMEM accumulator buffer
constexpr int kPfThreads = 320;
constexpr int kPfEpiThreads = 256;
// SMEM (after 1 KB alignment): [0, 96K) expand ring, 3 x 32 KB (B rows of a column tile; a rank > 128
// tile takes two stages, rank rows [0,128) and [128,r)); [96K, 224K) V (32 KB, 64 KB for rank > 128)
// then the staged y tiles (3, or 2 for rank > 128); the shrink ring spans all of [0, 224K) until D1 is
// done: 7 stages of 32 KB (x chunk 16 KB + A chunk <= 16 KB) or, for rank > 128, 4 of 48 KB.
constexpr int kPfStages = 3;           // expand-phase ring (B rows)
constexpr int kPfShrinkStages = 7;     // shrink-phase ring (at most)
constexpr int kPfStageBytes = 32768;
constexpr int kPfVBytes = 128 * 128 * 2;   // 32 KB: one V part of 128 tokens x 128 rank columns, bf16
constexpr int kPfYBytes = 128 * 128 * 2;   // one staged y tile (128 tokens x 128 columns, bf16)
constexpr int kPfYSlots = 3;               // staged y tiles in flight (at most)
constexpr int kPfBarBytes = 512;
constexpr int kPfSmem = 1024 /*align*/ + kPfStages * kPfStageBytes + 2 * kPfVBytes + 2 * kPfYBytes + kPfBarBytes;
static_assert(kPfSmem <= 232448, "prefill smem");
constexpr int kPfNTile = 128;          // expand columns per tile
constexpr int kPfTileWords = 8;        // per-tile record in the metadata blob

struct PrefillArgs {
    CUtensorMap tm_x;   // x [T][H_in], box {64, 128}, SW128
    CUtensorMap tm_a;   // A pages [n_pages+1][H_in], box {64, 1}, SW128 (gather4)
    CUtensorMap tm_b;   // B pages [n_pages+1][H_out], box {64, 1}, SW128 (gather4)
    CUtensorMap tm_y;   // y [T][H_out], box {64, 128}, SW128 (staged reads)
    CUtensorMap tm_y32; // y [T][H_out], box {64, 32}, SW128 (one epilogue warp's rows, TMA store)
    const char* box_maps;   // pool page arrays as 2D boxes {64, 8 << k} (A maps, then B maps), SW128
    int cs;                 // cluster size: the cs CTAs of a token tile split its shrink K and its columns
    float* pscratch;        // split-K partials [CTA][r/4 <= 64][128 rows][4] fp32 (L2-resident exchange)
    char* y;
    const int32_t* meta_global;
    unsigned long long* trace;
    int H_in, H_out, n_tiles, zero_page;
};

template <int W>
struct PfBlob {
    int32_t w[W];
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t pf_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void pf_bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void pf_arrive_tx(uint32_t bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void pf_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void pf_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_PFW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_PFW;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tm), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(dst),
        "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
// smem -> global tensor store (bulk group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tm), "r"(src),
                 "r"(c0), "r"(c1)
                 : "memory");
}
// ---- cluster split-K helpers
__device__ __forceinline__ uint32_t pf_cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t pf_mapa(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ void pf_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void pf_wait_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_PFWC:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_PFWC;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void pf_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D fp32, A/B bf16, M=128, N=n, B K-major (0) or MN-major (1)
__device__ __forceinline__ uint32_t umma_idesc(int n, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 lanes x 32 consecutive fp32 columns: thread i of the warp gets lane (base_lane + i), cols [col, col+32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
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
__device__ __forceinline__ unsigned long long pf_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ kernel
template <int W>
__global__ void __launch_bounds__(kPfThreads, 1)
    lora_prefill_tc_kernel(const __grid_constant__ PrefillArgs a, const __grid_constant__ PfBlob<W> blob) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = pf_smem(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;      // SW128 atoms need 1 KB alignment
    uint8_t* gbase = smem_raw + (base - raw);
    const uint32_t ring = base;                         // kPfStages x 32 KB
    const uint32_t vhi = base + kPfStages * kPfStageBytes;
    uint8_t* gv = gbase + kPfStages * kPfStageBytes;   // generic pointer to V
    const uint32_t bars = vhi + 2 * kPfVBytes + 2 * kPfYBytes;   // mbarriers + tmem slot
    // barriers: shrink ring full/empty [7] x 2, expand ring full/empty [3] x 2, then the rest
    auto full = [&](int s) { return bars + 8u * s; };
    auto empty = [&](int s) { return bars + 8u * (kPfShrinkStages + s); };
    auto full2 = [&](int s) { return bars + 8u * (2 * kPfShrinkStages + s); };
    auto empty2 = [&](int s) { return bars + 8u * (2 * kPfShrinkStages + kPfStages + s); };
    const uint32_t d1_full = bars + 8u * (2 * kPfShrinkStages + 2 * kPfStages);
    const uint32_t v_ready = d1_full + 8u;
    auto tm_full = [&](int b) { return v_ready + 8u + 8u * b; };
    auto tm_empty = [&](int b) { return v_ready + 24u + 8u * b; };
    auto y_full = [&](int b) { return v_ready + 40u + 8u * b; };
    auto y_empty = [&](int b) { return v_ready + 64u + 8u * b; };   // the 4 warps of the tile's group
    // split-K exchange (cs > 1): every peer's partial of the tile is in the L2 scratch
    const uint32_t pready = bars + 8u * (2 * kPfShrinkStages + 2 * kPfStages + 12);
    uint32_t* tmem_slot =
        reinterpret_cast<uint32_t*>(gbase + (bars + 8u * (2 * kPfShrinkStages + 2 * kPfStages + 13) - base));
    static_assert(8 * (2 * kPfShrinkStages + 2 * kPfStages + 13) + 4 <= kPfBarBytes, "barrier region");

    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile = blockIdx.x;
    const int32_t* rec = M + tile * kPfTileWords;
    const int tok0 = rec[0], nvalid = rec[1], r = rec[2], poff = rec[3];
    const float scale = __int_as_float(rec[4]);
    const int first_page = rec[5];   // >= 0: rank rows are pages [first_page, first_page + r)
    const int rp = (r + 15) & ~15;                      // rank padded to the MMA N/K granularity
    // v goes to the expand as bf16 (SURVEY §8(c) reading 4 allows it on the tcgen05 expand; rel-L2
    // budget in DESIGN.md); the y tiles are staged after it
    const bool wide = rp > 128;
    const int nys = wide ? 2 : 3;                                  // staged y slots
    const uint32_t yring = vhi + (wide ? 2u : 1u) * kPfVBytes;
    uint8_t* gy = gbase + (yring - base);
    const int nss = wide ? 4 : kPfShrinkStages;                    // shrink stages
    const uint32_t ssz = wide ? 49152u : 32768u;                   // shrink stage bytes
    const int nhalf = wide ? 2 : 1;                                // expand ring stages per column tile
    const int nkc_all = a.H_in / 64;                    // shrink K chunks of the tile
    const int cs = a.cs;
    const int ck = cs > 1 ? (int)pf_cluster_rank() : 0;  // this CTA's share of K: [kc_lo, kc_lo + nkc)
    const int kc_lo = ck * nkc_all / cs;
    const int nkc = (ck + 1) * nkc_all / cs - kc_lo;
    // expand column tiles of this CTA: [nt_lo, nt_lo + nnt) -- a tile's columns may be split over
    // several CTAs (each recomputes the tile's shrink) when the batch has fewer tiles than SMs
    const int nt_lo = rec[6];
    const int nnt = (rec[7] > 0 ? rec[7] : a.H_out / kPfNTile) - nt_lo;
    if (a.trace && tid == 0) a.trace[(size_t)tile * 4 + 0] = pf_gtime();

    if (tid == 0) {
        for (int s = 0; s < kPfShrinkStages; ++s) {
            pf_bar_init(full(s), 1);
            pf_bar_init(empty(s), 1);
        }
        for (int s = 0; s < kPfStages; ++s) {
            pf_bar_init(full2(s), 1);
            pf_bar_init(empty2(s), 1);
        }
        pf_bar_init(d1_full, 1);
        pf_bar_init(v_ready, (uint32_t)(kPfEpiThreads / 32 * cs));   // every epilogue warp of every CTA of the cluster
        pf_bar_init(pready, (uint32_t)cs);
        for (int b = 0; b < 2; ++b) {
            pf_bar_init(tm_full(b), 1);
            pf_bar_init(tm_empty(b), 128);
        }
        for (int b = 0; b < kPfYSlots; ++b) {   // slots [nys, 3) stay unused
            pf_bar_init(y_full(b), 1);
            pf_bar_init(y_empty(b), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // TMEM: D1 at columns [0,256), D2 buffers at [256,384) and [384,512)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(pf_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    if (cs > 1) pf_cluster_sync();   // every peer's barriers are initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // x and y may be produced by the preceding kernel in the stream
    if (tid == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ===================== TMA producer =====================
        int stage = 0;
        uint32_t phase = 0;
        const int ngr = rp / 4;   // gather4 groups (rank rows, padded with the zero page)
        // lane owns gather4 groups lane (rank rows [4 lane, 4 lane + 4)) and lane + 32 (rows 128 + ...)
        int pg[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = (lane + 32 * u) * 4 + q;
                pg[u][q] = j < r ? M[poff + j] : a.zero_page;
            }
        // contiguous adapters: the first rb = r & ~7 rank rows as 2D boxes of 128/64/32/16/8 rows
        // (one TMA request instead of rb/4 gather4s; the request rate bounded the rank-128 tiles).
        // Rows [rb, rp) come by gather4 with the pool's zero page past r, never from the pages
        // after the adapter's run (another tenant's rows, or freed ones: an Inf there would turn
        // 0 * B into NaN in this tenant's y)
        const bool use_box = first_page >= 0 && a.box_maps != nullptr;
        const int rb = use_box ? (r & ~7) : 0;
        // rank rows [row0, row1) of the run as boxes; row `row` lands at dst + (row - row0) * 128
        auto boxes = [&](uint32_t dst, int map_base, int col, uint32_t bar, int row0, int row1) {
            int row = row0;
            for (int k = 4; k >= 0; --k) {
                const int R = 8 << k;
                while (row1 - row >= R) {
                    tma_2d(dst + (uint32_t)(row - row0) * 128u,
                           reinterpret_cast<const CUtensorMap*>(a.box_maps + (map_base + k) * 128), col,
                           first_page + row, bar);
                    row += R;
                }
            }
        };
        // this lane's gather4 groups gi = lane + 32 u (rows 4 gi .. 4 gi + 3) not covered by the boxes
        const bool gat0 = lane >= rb / 4 && lane < ngr;
        const bool gat1 = lane + 32 >= rb / 4 && lane + 32 < ngr;
        for (int kq = 0; kq < nkc; ++kq) {
            const int kc = kc_lo + kq;
            pf_wait(empty(stage), phase ^ 1u);
            const uint32_t sb = ring + stage * ssz;
            if (lane == 0) {
                pf_arrive_tx(full(stage), (uint32_t)(128 * 128 + rp * 128));
                tma_2d(sb, &a.tm_x, kc * 64, tok0, full(stage));
                if (rb > 0) boxes(sb + 16384, 0, kc * 64, full(stage), 0, rb);
            }
            __syncwarp();
            if (gat0)
                tma_gather4(sb + 16384 + lane * 512, &a.tm_a, kc * 64, pg[0][0], pg[0][1], pg[0][2], pg[0][3], full(stage));
            if (gat1)
                tma_gather4(sb + 16384 + (lane + 32) * 512, &a.tm_a, kc * 64, pg[1][0], pg[1][1], pg[1][2], pg[1][3],
                            full(stage));
            if (++stage == nss) { stage = 0; phase ^= 1u; }
        }
        // the expand ring reuses shrink stages 0-2: wait until every shrink MMA has read them
        pf_wait(d1_full, 0);
        stage = 0;
        phase = 0;
        // expand: B rows of each 128-column tile, per ring stage the rank rows [128 hf, 128 hf + rh) of
        // half hf as MN-major SW128 atoms (8 rank rows x 64 cols): atom (kg, ng) at (ng * rh/8 + kg) * 1 KB;
        // a gather4 fills 4 rows of one atom
        for (int q = 0; q < nnt; ++q) {
            const int nt = nt_lo + q;
            // the y tile into slot q % nys once the group that had tile q - nys stored it
            if (lane == 0) {
                const int yb = q % nys;
                pf_wait(y_empty(yb), ((q / nys) & 1) ^ 1u);
                const uint32_t dst = yring + (uint32_t)yb * kPfYBytes;
                pf_arrive_tx(y_full(yb), (uint32_t)kPfYBytes);
                tma_2d(dst, &a.tm_y, nt * kPfNTile, tok0, y_full(yb));
                tma_2d(dst + kPfYBytes / 2, &a.tm_y, nt * kPfNTile + 64, tok0, y_full(yb));
            }
            for (int hf = 0; hf < nhalf; ++hf) {
                const int rh = min(128, rp - 128 * hf);
                pf_wait(empty2(stage), phase ^ 1u);
                const uint32_t sb = ring + stage * kPfStageBytes;
                if (lane == 0) {
                    pf_arrive_tx(full2(stage), (uint32_t)(rh * kPfNTile * 2));
                    const int b0 = 128 * hf, b1 = min(rb, 128 * hf + 128);
                    if (b1 > b0)
                        for (int h = 0; h < 2; ++h)
                            boxes(sb + (uint32_t)(h * (rh / 8)) * 1024u, kBoxKinds, nt * kPfNTile + h * 64, full2(stage), b0, b1);
                }
                __syncwarp();
                if (hf == 0 ? gat0 : gat1) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t dst = sb + (uint32_t)((h * (rh / 8) + (lane >> 1)) * 1024 + (lane & 1) * 512);
                        tma_gather4(dst, &a.tm_b, nt * kPfNTile + h * 64, pg[hf][0], pg[hf][1], pg[hf][2], pg[hf][3],
                                    full2(stage));
                    }
                }
                if (++stage == kPfStages) { stage = 0; phase ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one elected lane) =====================
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t id1 = umma_idesc(rp, 0);
        const uint32_t id2 = umma_idesc(kPfNTile, 1);
        for (int kc = 0; kc < nkc; ++kc) {
            pf_wait(full(stage), phase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t sb = ring + stage * ssz;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_f16(tmem, umma_desc(sb + kk * 32, 16, 1024), umma_desc(sb + 16384 + kk * 32, 16, 1024), id1,
                             (kc | kk) != 0);
                umma_commit(empty(stage));
                if (kc == nkc - 1) umma_commit(d1_full);
            }
            __syncwarp();
            if (++stage == nss) { stage = 0; phase ^= 1u; }
        }
        stage = 0;
        phase = 0;
        pf_wait_cluster(v_ready, 0);
        tc_fence_after();
        for (int q = 0; q < nnt; ++q) {
            const int b = q & 1;
            pf_wait(tm_empty(b), ((q >> 1) & 1) ^ 1u);
            for (int hf = 0; hf < nhalf; ++hf) {
                const int rh = min(128, rp - 128 * hf);
                pf_wait(full2(stage), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sb = ring + stage * kPfStageBytes;
                    const uint32_t dcol = tmem + 256u + 128u * b;
                    const uint32_t lbo = (uint32_t)(rh / 8) * 1024u;   // MN-direction atom stride
                    for (int ks = 0; ks < rh / 16; ++ks) {
                        const int kg = 8 * hf + ks;   // k-step over the whole rank
                        const uint32_t voff = (uint32_t)(kg >> 2) * 16384u + (uint32_t)(kg & 3) * 32u;
                        const uint64_t bd = umma_desc(sb + (uint32_t)ks * 2048u, lbo, 1024);
                        umma_f16(dcol, umma_desc(vhi + voff, 16, 1024), bd, id2, kg != 0);
                    }
                    umma_commit(empty2(stage));
                    if (hf == nhalf - 1) umma_commit(tm_full(b));
                }
                __syncwarp();
                if (++stage == kPfStages) { stage = 0; phase ^= 1u; }
            }
        }
    } else {
        // ===================== epilogue: group eg = warps 2+4eg .. 5+4eg; warp w -> TMEM lanes 32*(w%4) .. +32
        const int eg = (warp - 2) >> 2;
        const int etid = tid - 64;   // 0 .. 255
        const int sub = warp & 3;
        const int row = sub * 32 + lane;   // token row within the tile
        const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
        // ---- v = s * D1 -> bf16 (the expand's A operand); the two groups take alternate 32-column chunks
        pf_wait(d1_full, 0);
        tc_fence_after();
        if (a.trace && tid == 64) a.trace[(size_t)tile * 4 + 2] = pf_gtime();
        // the bf16 v chunk (8 columns c8*8.. of token row rr) at its K-major SW128 slot: atom kk = cols
        // [64kk, 64kk+64), row at (rr/8)*1024 + (rr%8)*128 inside the 16 KB atom, 16-B chunk c at c ^ (rr%8)
        auto v_off = [](int rr, int col) -> uint32_t {
            const int kk = col >> 6, chunk = (col & 63) >> 3;
            return (uint32_t)kk * 16384u + (uint32_t)(rr >> 3) * 1024u + (uint32_t)(rr & 7) * 128u +
                   (uint32_t)((chunk ^ (rr & 7)) * 16);
        };
        auto pack8 = [&](const float* f, int col) -> uint4 {   // s * D1 -> bf16; columns >= r are exact zeros
            uint32_t hw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float f0 = col + 2 * e < r ? f[2 * e] * scale : 0.f;
                const float f1 = col + 2 * e + 1 < r ? f[2 * e + 1] * scale : 0.f;
                __nv_bfloat162 h = __floats2bfloat162_rn(f0, f1);
                hw[e] = *reinterpret_cast<uint32_t*>(&h);
            }
            return make_uint4(hw[0], hw[1], hw[2], hw[3]);
        };
        if (cs > 1) {
            // split-K: this CTA's D1 is a partial over its K share.  (1) every CTA writes its partial to an
            // L2-resident scratch as float4 column quads [CTA][col/4][row][4] (a warp's 32 rows = 512
            // coalesced bytes per quad); (2) once every peer's partial is released (remote mbarrier arrive, cluster scope),
            // CTA ck reduces the rows [ck*128/cs, (ck+1)*128/cs) over the cs partials in rank order
            // (deterministic), scales and rounds them to bf16 and (3) writes those v rows into the V
            // buffer of every CTA of the cluster (DSMEM), whose v_ready then counts the peers' warps.
            float4* pmine = reinterpret_cast<float4*>(a.pscratch) + (size_t)blockIdx.x * (kPfMaxRank / 4) * 128 + row;
            for (int c0 = 32 * eg; c0 < rp; c0 += 64) {
                float v[32];
                tmem_ld32(tmem + lane_addr + (uint32_t)c0, v);
                const int nq = rp - c0 < 32 ? (rp - c0) / 4 : 8;   // rp % 16 == 0
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (i < nq) pmine[(size_t)(c0 / 4 + i) * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (etid == 0)
                for (int c = 0; c < cs; ++c) pf_arrive_remote(pf_mapa(pready, (uint32_t)c));
            pf_wait_cluster(pready, 0);
            const int r_lo = ck * 128 / cs, nrows = (ck + 1) * 128 / cs - r_lo;
            const float4* part0 = reinterpret_cast<const float4*>(a.pscratch) + (size_t)(blockIdx.x - ck) * (kPfMaxRank / 4) * 128;
            for (int it = etid; it < nrows * (rp / 8); it += kPfEpiThreads) {
                const int rr = r_lo + it % nrows, c8 = it / nrows;
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = 0.f;
                for (int c = 0; c < cs; ++c) {
                    const float4* src = part0 + (size_t)c * (kPfMaxRank / 4) * 128 + (size_t)(c8 * 2) * 128 + rr;
                    const float4 g0 = __ldcg(src), g1 = __ldcg(src + 128);
                    f[0] += g0.x; f[1] += g0.y; f[2] += g0.z; f[3] += g0.w;
                    f[4] += g1.x; f[5] += g1.y; f[6] += g1.z; f[7] += g1.w;
                }
                const uint4 w = pack8(f, c8 * 8);
                const uint32_t dst = vhi + v_off(rr, c8 * 8);
                for (int c = 0; c < cs; ++c)
                    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(pf_mapa(dst, (uint32_t)c)),
                                 "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                                 : "memory");
            }
            asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");   // generic -> tensor-core reads
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            __syncwarp();
            // A CTA cannot retire before all DSMEM traffic into it is done: its MMA warp waits for its
            // v_ready, which completes only after every peer warp's release-arrive that follows that
            // warp's stores (and pready likewise), and the CTA exits after a __syncthreads with the MMA
            // warp.  (compute-sanitizer racecheck does not follow mbarriers across the cluster and
            // reports these stores as "into a block that might have already exited"; an explicit
            // exit-time barrier.cluster hangs under racecheck and measured 0.5-1 % slower natively.)
            if (lane == 0)
                for (int c = 0; c < cs; ++c) pf_arrive_remote(pf_mapa(v_ready, (uint32_t)c));
        } else {
            for (int c0 = 32 * eg; c0 < rp; c0 += 64) {
                float v[32];
                tmem_ld32(tmem + lane_addr + (uint32_t)c0, v);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<uint4*>(gv + v_off(row, c0 + q * 8)) = pack8(v + q * 8, c0 + q * 8);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor-core reads
            tc_fence_before();
            __syncwarp();
            if (lane == 0) pf_arrive(v_ready);
        }
        if (a.trace && tid == 64) a.trace[(size_t)tile * 4 + 3] = pf_gtime();
        // ---- expand tiles q = eg, eg + 2, ...: y[row][n0 .. n0+128) += D2 (one rounding) in the staged
        //      y tile (the producer loads it by TMA into slot q % 3; SW128: row at (row/8)*1024 +
        //      (row%8)*128 per 64-column half, 16-B chunk c at c ^ (row%8)).  A warp whose 32 rows are all
        //      in the segment stores them by TMA; a warp holding rows past the segment (they belong to
        //      other segments' tiles) stores its valid rows with STG.
        const bool valid = row < nvalid;
        const bool warp_full = sub * 32 + 32 <= nvalid;
        for (int q = eg; q < nnt; q += 2) {
            const int nt = nt_lo + q;
            const int b = eg;   // TMEM buffer q & 1
            pf_wait(tm_full(b), (q >> 1) & 1);
            const int yb = q % nys;
            pf_wait(y_full(yb), (q / nys) & 1);
            tc_fence_after();
            uint8_t* ys = gy + yb * kPfYBytes + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll 1
            for (int c0 = 0; c0 < kPfNTile; c0 += 32) {
                float d[32];
                tmem_ld32(tmem + lane_addr + 256u + 128u * b + (uint32_t)c0, d);
                if (valid) {
                    uint4 o4[4];
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const int col = c0 + q4 * 8;
                        const int h = col >> 6, chunk = (col & 63) >> 3;
                        const uint4 yv = *reinterpret_cast<const uint4*>(ys + h * (kPfYBytes / 2) + ((chunk ^ (row & 7)) << 4));
                        const uint32_t w[4] = {yv.x, yv.y, yv.z, yv.w};
                        uint32_t o[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float lo = __uint_as_float(w[e] << 16) + d[q4 * 8 + 2 * e];
                            const float hi = __uint_as_float(w[e] & 0xffff0000u) + d[q4 * 8 + 2 * e + 1];
                            __nv_bfloat162 hb = __floats2bfloat162_rn(lo, hi);
                            o[e] = *reinterpret_cast<uint32_t*>(&hb);
                        }
                        o4[q4] = make_uint4(o[0], o[1], o[2], o[3]);
                    }
                    // back into the row's own (swizzled) slots of the staged tile
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const int col = c0 + q4 * 8;
                        const int h = col >> 6, chunk = (col & 63) >> 3;
                        *reinterpret_cast<uint4*>(ys + h * (kPfYBytes / 2) + ((chunk ^ (row & 7)) << 4)) = o4[q4];
                    }
                }
            }
            tc_fence_before();
            pf_arrive(tm_empty(b));
            const uint32_t yslot_s = yring + (uint32_t)yb * kPfYBytes;
            if (warp_full) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // STS -> TMA store reads
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&a.tm_y32, yslot_s + (uint32_t)sub * 4096u, nt * kPfNTile, tok0 + sub * 32);
                    tma_store_2d(&a.tm_y32, yslot_s + kPfYBytes / 2 + (uint32_t)sub * 4096u, nt * kPfNTile + 64,
                                 tok0 + sub * 32);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // slot may be refilled
                    pf_arrive(y_empty(yb));
                }
            } else {
                // the warp's valid rows as 256-B row segments, two rows per STG.128 instruction
                __syncwarp();
                const uint8_t* yslot = gy + yb * kPfYBytes;
#pragma unroll 4
                for (int i = 0; i < 16; ++i) {
                    const int rr = sub * 32 + i * 2 + (lane >> 4), c16 = lane & 15;
                    if (rr < nvalid) {
                        const uint4 v = *reinterpret_cast<const uint4*>(
                            yslot + (c16 >> 3) * (kPfYBytes / 2) + (rr >> 3) * 1024 + (rr & 7) * 128 +
                            (((c16 & 7) ^ (rr & 7)) << 4));
                        *reinterpret_cast<uint4*>(a.y + ((size_t)(tok0 + rr) * a.H_out + nt * kPfNTile + c16 * 8) * 2) = v;
                    }
                }
                __syncwarp();
                if (lane == 0) pf_arrive(y_empty(yb));
            }
        }
        // the TMA stores are complete (not just read) before the CTA retires
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
    if (a.trace && tid == 0) a.trace[(size_t)tile * 4 + 1] = pf_gtime();
}

// ------------------------------------------------------------------ host side
bool prefill_supported(int H_in, int H_out, int esz) {
    return esz == 2 && H_in % 64 == 0 && H_out % kPfNTile == 0 && H_in >= 64;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2D bf16 tensor map [rows][cols] with a {64, box_rows} SWIZZLE_128B box
int make_tmap_bf16(void* tm_out, const void* base, int64_t rows, int64_t cols, int box_rows) {
    auto enc = get_encode();
    if (!enc) return (int)cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(tm_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

int make_box_tmaps(void* host_out, const void* dA, const void* dB, int n_rows, int H_in, int H_out) {
    char* o = static_cast<char*>(host_out);
    for (int k = 0; k < kBoxKinds; ++k) {
        if (make_tmap_bf16(o + k * 128, dA, n_rows, H_in, 8 << k)) return 1;
        if (make_tmap_bf16(o + (kBoxKinds + k) * 128, dB, n_rows, H_out, 8 << k)) return 1;
    }
    return 0;
}

template <int W>
static cudaError_t launch_pf(const PrefillArgs& a, const Plan& pl, cudaStream_t st) {
    // cudaFuncSetAttribute is per device: one bit per device
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;
    if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(lora_prefill_tc_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kPfSmem);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    PfBlob<W> blob;
    if (W > 1)
        for (size_t i = 0; i < pl.pf_blob.size(); ++i) blob.w[i] = pl.pf_blob[i];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.n_pf_tiles);
    cfg.blockDim = dim3(kPfThreads);
    cfg.dynamicSmemBytes = kPfSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = a.cs > 1 ? a.cs : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, lora_prefill_tc_kernel<W>, a, blob);
}

int launch_prefill(const Plan& pl, const PrefillLaunch& L, cudaStream_t st, int* launches) {
    PrefillArgs a;
    std::memset(&a, 0, sizeof(a));
    int e = make_tmap_bf16(&a.tm_x, L.x, L.T, L.H_in, 128);
    if (e) return e;
    std::memcpy(&a.tm_a, L.tm_a, sizeof(CUtensorMap));
    std::memcpy(&a.tm_b, L.tm_b, sizeof(CUtensorMap));
    a.box_maps = static_cast<const char*>(L.box_maps);
    e = make_tmap_bf16(&a.tm_y, L.y, L.T, L.H_out, 128);
    if (e) return e;
    e = make_tmap_bf16(&a.tm_y32, L.y, L.T, L.H_out, 32);
    if (e) return e;
    a.y = static_cast<char*>(L.y);
    a.meta_global = L.meta_dev;
    a.trace = L.trace;
    a.H_in = L.H_in;
    a.H_out = L.H_out;
    a.n_tiles = pl.n_pf_tiles;
    a.cs = pl.pf_cs > 1 ? pl.pf_cs : 1;
    a.pscratch = L.pscratch;
    if (a.cs > 1 && !a.pscratch) return (int)cudaErrorInvalidValue;
    a.zero_page = L.zero_page;
    const size_t n = pl.pf_blob.size();
    cudaError_t r;
    if (n <= 2048) r = launch_pf<2048>(a, pl, st);
    else if (n <= 7680) r = launch_pf<7680>(a, pl, st);
    else return (int)cudaErrorNotSupported;   // planner caps prefill work to the parameter blob
    *launches += 1;
    return (int)r;
}

}  // namespace lora
