// fused_base_kernel.cu -- SURVEY §8(f) NEXT row 2: the LoRA delta fused into the base projection
// GEMM (§4.1: "incorporate the operators of GPU LoRA computation into the base
// LLM inference process"; Eq. 1: y = x·W + x·A·B, with the per-adapter scale s).
//
// One CTA per (128-token tile of one segment, NT-column tile of y; NT = 256, or 128 when
// H_out % 256 != 0), column tiles the fast grid dimension so a token tile's CTAs share x in L2:
//     D_base[t][n]  = Σ_k X[t][k] · W[k][n]          base GEMM, TMEM columns [0, NT)
//     D1[t][j]      = Σ_k X[t][k] · A_g[k][j]        shrink,    TMEM columns [NT, NT + r16)
//     D_base[t][n] += Σ_j bf16(s_g·D1[t][j]) · B_g[j][n]   expand into the base accumulator
//     y[t][n]       = bf16(D_base[t][n])             one rounding, y written once
// Each K stage's x chunk feeds both the base MMA and the shrink MMA, so x is read once for both
// and y is never read: the separate delta pass's y read + write disappear.
// First version: the shrink is recomputed per column tile (r16/NT extra MMA work), tiles never
// span segments, and rank <= 128 (the N2 limits).  The ring holds 3-4 stages sized by the tile's
// rank.  Layouts are N2's (prefill_kernel.cu): x box {64,128} SW128 K-major; A / B rank rows as 2D
// boxes when the adapter's pages are one run, else tile::gather4; B and W tiles MN-major SW128
// atoms (8 K-rows x 64 columns); V K-major SW128.  Measurements: DESIGN.md §10.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstring>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

constexpr int kFbThreads = 192;        // warp 0: TMA producer, warp 1: MMA issuer, warps 2-5: epilogue
constexpr int kFbMaxStages = 4;   // the ring holds as many stages as fit (3 or 4, by the tile's rank)
// ring stage: X chunk 16 KB + W chunk (64 x NT columns) + A chunk <= 16 KB; after the mainloop
// stage 0 holds the expand's B tile (r16 <= 128 rank rows x NT columns <= 64 KB)
constexpr int fb_stage_bytes(int nt) { return 16384 + nt * 128 + 16384; }
// V: 128 tokens x r16 <= 128, bf16, K-major SW128 (32 KB), in a ring stage after the mainloop
constexpr int kFbSmem = 227 * 1024;                  // the whole opt-in maximum: the ring takes what the rank allows
constexpr int kFbRingBytes = kFbSmem - 1024 - 256;   // minus alignment slack and the barrier block
constexpr int kFbTileWords = 8;
static_assert(3 * fb_stage_bytes(256) <= kFbRingBytes, "three stages at rank 128");

struct FusedBaseArgs {
    CUtensorMap tm_x;   // x [T][H_in], box {64, 128}
    CUtensorMap tm_w;   // W [H_in][H_out], box {64, 64}
    CUtensorMap tm_a;   // A pages [n_pages+1][H_in], box {64, 1} (gather4)
    CUtensorMap tm_b;   // B pages [n_pages+1][H_out], box {64, 1} (gather4)
    const char* box_maps;   // the pool's page arrays as 2D boxes {64, 8 << k} (A maps, then B maps), or null
    char* y;
    int H_in, H_out, zero_page;
    int ring_bytes;   // dynamic shared memory for the ring (the launch's smem minus 1280 B)
};

struct FbBlob {
    int32_t w[kFusedBaseMaxWords];   // [n_tiles][8] {tok0, nvalid, rank, page_off, scale_bits}, then pages
};

namespace {
__device__ __forceinline__ uint32_t fb_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void fb_bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fb_arrive_tx(uint32_t bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void fb_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fb_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_FBW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_FBW;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fb_tma_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tm), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void fb_gather4(uint32_t dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                           uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(dst),
        "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1 (sm_100)
__device__ __forceinline__ uint64_t fb_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D fp32, A/B bf16, M=128, N=n, B K-major (0) or MN-major (1)
__device__ __forceinline__ uint32_t fb_idesc(int n, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void fb_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void fb_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fb_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fb_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fb_ld32(uint32_t taddr, float (&v)[32]) {
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

template <int NT>   // output columns per CTA (128 or 256 = the MMA N of the base GEMM)
__global__ void __launch_bounds__(kFbThreads, 1)
    lora_fused_base_kernel(const __grid_constant__ FusedBaseArgs a, const __grid_constant__ FbBlob blob) {
    // stage = X 16 KB + W (64 x NT) + A (r16 rows x 128 B): 4 stages fit up to rank 64 at NT = 256
    constexpr uint32_t kTmemCols = NT == 256 ? 512u : 256u;   // D_base [0, NT), D1 [NT, NT + 128)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = fb_smem(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    const uint32_t ring = base;
    const uint32_t bars = base + (uint32_t)a.ring_bytes;
    auto full = [&](int s) { return bars + 8u * s; };
    auto empty = [&](int s) { return bars + 8u * (kFbMaxStages + s); };
    const uint32_t d_full = bars + 8u * (2 * kFbMaxStages);
    const uint32_t v_ready = d_full + 8u;
    const uint32_t b_full = d_full + 16u;
    const uint32_t d2_full = d_full + 24u;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (d_full + 32u - base));
    static_assert(8 * (2 * kFbMaxStages + 4) + 4 <= 256, "barrier block");

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // grid: x = column tile (fast), y = token tile -- a token tile's column CTAs run together and
    // share its x tiles through L2 (W stays L2-resident); the transposed order re-streams x from HBM
    // once per column tile
    const int32_t* rec = blob.w + blockIdx.y * kFbTileWords;
    const int tok0 = rec[0], nvalid = rec[1], r = rec[2], poff = rec[3];
    const int first_page = rec[5];   // >= 0: the rank rows are pages [first_page, first_page + r)
    const float scale = __int_as_float(rec[4]);
    const int rp = r > 0 ? (r + 15) & ~15 : 0;
    const int n0 = blockIdx.x * NT;
    const int nkc = a.H_in / 64;
    const uint32_t kStage = (uint32_t)(16384 + NT * 128 + rp * 128);   // multiple of 2 KB
    const int nst = min(kFbMaxStages, (int)((uint32_t)a.ring_bytes / kStage));
    // after the mainloop: the expand's B tile goes into the ring stage the producer would fill next
    // (nkc % nst, the first one released, so its load overlaps the last stages' MMAs) and V into the
    // one after it (free once every mainloop MMA has completed)
    const uint32_t bbuf = ring + (uint32_t)(nkc % nst) * kStage;
    const uint32_t vbuf = ring + (uint32_t)((nkc + 1) % nst) * kStage;
    uint8_t* gv = gbase + (vbuf - base);

    if (tid == 0) {
        for (int s = 0; s < kFbMaxStages; ++s) {
            fb_bar_init(full(s), 1);
            fb_bar_init(empty(s), 1);
        }
        fb_bar_init(d_full, 1);
        fb_bar_init(v_ready, 128);
        fb_bar_init(b_full, 1);
        fb_bar_init(d2_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // TMEM: D_base at columns [0, NT), D1 at [NT, NT + 128)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(fb_smem(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fb_fence_before();
    __syncthreads();
    fb_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        const int ngr = rp / 4;
        // contiguous adapters: the first rb = r & ~7 rank rows as 2D boxes of 128/64/32/16/8 rows
        // (one TMA request instead of rb/4 gather4s); rows [rb, rp) by gather4 with the pool's zero
        // page past r -- never the pages after the adapter's run (another tenant's or freed rows,
        // where an Inf would turn 0 * B into NaN)
        const bool use_box = first_page >= 0 && a.box_maps != nullptr;
        const int rb = use_box ? (r & ~7) : 0;
        const bool gat = lane >= rb / 4 && lane < ngr;
        auto boxes = [&](uint32_t dst, int map_base, int col, uint32_t bar) {
            int row = 0;
            for (int k = 4; k >= 0; --k) {
                const int R = 8 << k;
                while (rb - row >= R) {
                    fb_tma_2d(dst + (uint32_t)row * 128u,
                              reinterpret_cast<const CUtensorMap*>(a.box_maps + (map_base + k) * 128), col,
                              first_page + row, bar);
                    row += R;
                }
            }
        };
        int pg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = lane * 4 + q;
            pg[q] = j < r ? blob.w[poff + j] : a.zero_page;
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int kc = 0; kc < nkc; ++kc) {
            fb_wait(empty(stage), phase ^ 1u);
            const uint32_t sb = ring + stage * kStage;
            if (lane == 0) {
                fb_arrive_tx(full(stage), (uint32_t)(16384 + NT * 128 + rp * 128));
                fb_tma_2d(sb, &a.tm_x, kc * 64, tok0, full(stage));
                // W rows [64kc, 64kc+64) x columns [n0, n0+NT): NT/64 MN-major atom columns of 8 KB
#pragma unroll
                for (int h = 0; h < NT / 64; ++h) fb_tma_2d(sb + 16384 + h * 8192, &a.tm_w, n0 + h * 64, kc * 64, full(stage));
                if (rb > 0) boxes(sb + 16384 + NT * 128, 0, kc * 64, full(stage));
            }
            __syncwarp();
            if (gat)
                fb_gather4(sb + 16384 + NT * 128 + lane * 512, &a.tm_a, kc * 64, pg[0], pg[1], pg[2], pg[3], full(stage));
            if (++stage == nst) { stage = 0; phase ^= 1u; }
        }
        if (r > 0) {   // the expand's B tile into the next ring stage, once its last mainloop MMAs are done
            fb_wait(empty(stage), phase ^ 1u);
            if (lane == 0) {
                fb_arrive_tx(b_full, (uint32_t)(rp * NT * 2));
                if (rb > 0)
                    for (int h = 0; h < NT / 64; ++h)
                        boxes(bbuf + (uint32_t)(h * (rp / 8)) * 1024u, kBoxKinds, n0 + h * 64, b_full);
            }
            __syncwarp();
            if (gat)
#pragma unroll
                for (int h = 0; h < NT / 64; ++h) {
                    const uint32_t dst = bbuf + (uint32_t)((h * (rp / 8) + (lane >> 1)) * 1024 + (lane & 1) * 512);
                    fb_gather4(dst, &a.tm_b, n0 + h * 64, pg[0], pg[1], pg[2], pg[3], b_full);
                }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        const uint32_t id_base = fb_idesc(NT, 1);
        const uint32_t id1 = rp > 0 ? fb_idesc(rp, 0) : 0u;
        int stage = 0;
        uint32_t phase = 0;
        for (int kc = 0; kc < nkc; ++kc) {
            fb_wait(full(stage), phase);
            fb_fence_after();
            if (lane == 0) {
                const uint32_t sb = ring + stage * kStage;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t xd = fb_desc(sb + kk * 32, 16, 1024);
                    fb_mma(tmem, xd, fb_desc(sb + 16384 + kk * 2048, 8192, 1024), id_base, (kc | kk) != 0);
                    if (rp > 0)
                        fb_mma(tmem + (uint32_t)NT, xd, fb_desc(sb + 16384 + NT * 128 + kk * 32, 16, 1024), id1, (kc | kk) != 0);
                }
                fb_commit(empty(stage));
                if (kc == nkc - 1) fb_commit(d_full);
            }
            __syncwarp();
            if (++stage == nst) { stage = 0; phase ^= 1u; }
        }
        if (rp > 0) {
            fb_wait(v_ready, 0);
            fb_wait(b_full, 0);
            fb_fence_after();
            if (lane == 0) {
                const uint32_t lbo = (uint32_t)(rp / 8) * 1024u;
                for (int ks = 0; ks < rp / 16; ++ks) {
                    const uint32_t voff = (uint32_t)(ks >> 2) * 16384u + (uint32_t)(ks & 3) * 32u;
                    fb_mma(tmem, fb_desc(vbuf + voff, 16, 1024), fb_desc(bbuf + (uint32_t)ks * 2048u, lbo, 1024), id_base, 1u);
                }
            }
        }
        if (lane == 0) fb_commit(d2_full);
        __syncwarp();
    } else {
        // ===================== epilogue: warps 2..5 -> TMEM lanes 32*(warp%4) .. +32 =====================
        const int sub = warp & 3;
        const int row = sub * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
        if (rp > 0) {
            // V = s · D1 -> bf16, K-major SW128 (atom kk = columns [64kk, 64kk+64)); columns >= r are 0
            fb_wait(d_full, 0);
            fb_fence_after();
            for (int c0 = 0; c0 < rp; c0 += 32) {
                float v[32];
                fb_ld32(tmem + lane_addr + (uint32_t)NT + (uint32_t)c0, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t hw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j0 = c0 + q * 8 + 2 * e;
                        const float f0 = j0 < r ? v[q * 8 + 2 * e] * scale : 0.f;
                        const float f1 = j0 + 1 < r ? v[q * 8 + 2 * e + 1] * scale : 0.f;
                        __nv_bfloat162 h = __floats2bfloat162_rn(f0, f1);
                        hw[e] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    const int col = c0 + q * 8;
                    const int kk = col >> 6, chunk = (col & 63) >> 3;
                    const uint32_t off = (uint32_t)kk * 16384u + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u +
                                         (uint32_t)((chunk ^ (row & 7)) * 16);
                    *reinterpret_cast<uint4*>(gv + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor-core reads
            fb_fence_before();
            fb_arrive(v_ready);
        }
        // y[tok0 + row][n0 .. n0+NT) = bf16(D_base): valid rows only (rows past the segment belong
        // to other tiles).  Each 32-column chunk of the warp's 32 rows is staged in the (now idle)
        // ring, 64 B per row with its four 16-B pieces rotated by row (bank spread), then leaves as
        // 8 rows x 64 contiguous bytes per store instruction instead of 32 rows x 16 B.
        fb_wait(d2_full, 0);
        fb_fence_after();
        uint8_t* stg = gbase + (ring - base) + sub * 2048;
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 32) {
            float d[32];
            fb_ld32(tmem + lane_addr + (uint32_t)c0, d);
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
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = i * 32 + lane, rr = idx >> 2, qq = idx & 3;
                const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * 64 + ((qq + rr) & 3) * 16);
                if (sub * 32 + rr < nvalid)
                    *reinterpret_cast<uint4*>(a.y + ((size_t)(tok0 + sub * 32 + rr) * a.H_out + n0 + c0 + qq * 8) * 2) = v;
            }
            __syncwarp();
        }
    }
    fb_fence_before();
    __syncthreads();
    if (warp == 1) {
        fb_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

int make_tmap_bf16(void* tm_out, const void* base, int64_t rows, int64_t cols, int box_rows);   // prefill_kernel.cu

int launch_fused_base(const FusedBaseLaunch& L, const int32_t* words, int n_words, int n_tiles, lora_cuda_stream st) {
    if (n_words > kFusedBaseMaxWords || n_tiles <= 0) return (int)cudaErrorInvalidValue;
    FusedBaseArgs a;
    std::memset(&a, 0, sizeof(a));
    int e = make_tmap_bf16(&a.tm_x, L.x, L.T, L.H_in, 128);
    if (!e) e = make_tmap_bf16(&a.tm_w, L.w, L.H_in, L.H_out, 64);
    if (e) return e;
    std::memcpy(&a.tm_a, L.tm_a, sizeof(CUtensorMap));
    std::memcpy(&a.tm_b, L.tm_b, sizeof(CUtensorMap));
    a.box_maps = static_cast<const char*>(L.box_maps);
    a.y = static_cast<char*>(L.y);
    a.H_in = L.H_in;
    a.H_out = L.H_out;
    a.zero_page = L.zero_page;
    FbBlob blob;   // the kernel-parameter blob (copied into the launch)
    std::memcpy(blob.w, words, (size_t)n_words * 4);
    // cudaFuncSetAttribute is per device: one bit per device
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return (int)cudaErrorInvalidDevice;
    const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;
    if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
        cudaError_t ce = cudaFuncSetAttribute(lora_fused_base_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFbSmem);
        if (ce == cudaSuccess)
            ce = cudaFuncSetAttribute(lora_fused_base_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFbSmem);
        if (ce != cudaSuccess) return (int)ce;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    a.ring_bytes = kFbRingBytes;
    if (L.H_out % 256 == 0)
        lora_fused_base_kernel<256><<<dim3(L.H_out / 256, n_tiles), kFbThreads, kFbSmem, st>>>(a, blob);
    else
        lora_fused_base_kernel<128><<<dim3(L.H_out / 128, n_tiles), kFbThreads, kFbSmem, st>>>(a, blob);
    return (int)cudaGetLastError();
}

}  // namespace lora
