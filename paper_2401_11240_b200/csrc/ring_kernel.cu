// ring_kernel.cu -- N1r: the persistent ring pair for bf16 decode applies, sm_100a.
//
// Computes the same delta as the PDL pair of decode_kernel.cu (§2.1 Eq. 1, P:276-280;
// MBGMV semantics, no padding to the batch's max rank):
//     v_t[j]  = Σ_k x_t[k] · A_g[j][k]                   shrink (fp32 accumulate, k-slice partials)
//     y_t[n] += s_g · Σ_j v_t[j] · B_g[j][n]             expand (fp32 accumulate, one rounding)
// with the same arithmetic (bf16 mma.sync m16n8k16, v split into bf16 hi + lo, k-slice partials
// summed in slice order), so its results are bitwise equal to the pair's.
//
// Why another pair (DESIGN.md §6 N1r).  The pair launches one CTA per 32 KB work unit.  A c2 q/k/v
// apply has 768 shrink + 768 expand units; SMEM (and, for the expand, the register file) holds
// ~4-5 units per SM, so the expand grid ran in two waves whose second wave fetched its B rows only
// after the first wave's CTAs exited -- the HBM latency of those rows sat on the critical path.
// Here each kernel runs ONE persistent CTA per SM that streams its list of 32 KB tiles through a
// ring of SMEM stages (a producer warp issuing cp.async.bulk, 2 KB row pieces, mbarrier tx
// counts), so the next tile's rows are always in flight while the consumers compute:
//   * both kernels fill their rings BEFORE griddepcontrol.wait (adapter pages are immutable), and
//     trigger launch_dependents at once, so the expand CTAs stream B while the shrink computes and
//     the next apply's shrink CTAs stream A while this expand computes;
//   * one shrink CTA + one expand CTA fit an SM together (the launcher sizes the rings so), and the
//     host assigns tiles to CTAs longest-first (LPT) so every SM gets the same bytes.
// Shrink tile = (gc, k-slice of 1024, 16 rank rows) = 32 KB of A; expand unit = (gc, 1024-column
// slice), processed as ceil(r/16) tiles of 16 B rows x 1024 columns (32 KB), accumulated in
// registers, y added once after the unit's last tile.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "decode_common.cuh"
#include "kernel_config.h"
#include "plan.h"

namespace lora {

constexpr int kRingWarps = 8;                                  // consumer warps
constexpr int kRingThreads = kRingWarps * 32;                  // shrink: consumers only
constexpr int kRingEThreads = (kRingWarps + 4) * 32;           // expand: + producer, loader, 2 idle warps
constexpr int kRingConsumers = kRingWarps * 32;
constexpr int kRingMaxStages = 6;
constexpr int kSPitch = kKSlice * 2 + 64;                      // A row pitch: rows g, g+1 16 banks apart
constexpr int kSStageA = kShrinkRowsMma * kSPitch;             // 33,792 B of A rows; x rows follow
constexpr int kSPartOff = 128;                                 // part sums [2][8 warps][16 rows][8 tokens] fp32
constexpr int kSRingOff = kSPartOff + 2 * kRingWarps * 16 * 8 * 4;   // 8,320
constexpr int kECols = 1024;                                   // columns per expand unit
constexpr int kEPitch = kECols * 2 + 16;                       // B / y row pitch (conflict-free ldmatrix)
constexpr int kEStage = 16 * kEPitch;                          // 33,024 B
constexpr int kSmemPerSM = 228 * 1024;                         // sm_100: shared memory per SM
constexpr int kSmemReserved = 1024;                            // per resident CTA
// a shrink CTA larger than this cannot share an SM with another shrink CTA
constexpr int kSMinSmem = kSmemPerSM / 2 - kSmemReserved + 16;

struct RingArgs {
    DecodeJob jobs[kMaxJobs];
    float* vbuf;
    const int32_t* meta_global;   // blob in device memory (too large for the parameters) or null
    unsigned long long* trace;    // optional per-CTA timestamps [cta][64]
    int list_off;                 // blob word offset: per-CTA tile offsets [n_cta + 1], then the tile words
    int n_cta;
    int ns;                       // ring stages
    int s_stage;                  // shrink stage bytes: 16 A rows + the launch's max tokens of x rows
    int e_vpitch, e_voff, e_yoff, e_ybuf, e_ringoff;   // expand smem layout (bytes)
};

// tile words.  shrink: gc | ks << 15 | jb << 20.  expand: gc | cs << 15 | jb << 20 | first << 24 | last << 25
__device__ __forceinline__ int tw_gc(int w) { return w & 0x7fff; }
__device__ __forceinline__ int tw_a(int w) { return (w >> 15) & 0x1f; }
__device__ __forceinline__ int tw_jb(int w) { return (w >> 20) & 0xf; }
__device__ __forceinline__ bool tw_first(int w) { return (w >> 24) & 1; }
__device__ __forceinline__ bool tw_last(int w) { return (w >> 25) & 1; }
__device__ __forceinline__ int gcf(const int32_t* M, int gc, int f) { return M[kHdrWords + gc * kGcFields + f]; }
__device__ __forceinline__ int pg_at(const int32_t* M, int ref, int j) { return ref >= 0 ? M[ref + j] : (~ref) + j; }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float4 ldg_cg_f4(const float* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kRingConsumers) : "memory"); }

// ------------------------------------------------------------------ shrink
// Placement (measured, scripts/coresidency_probe.cu): a warp's registers come from its SM
// sub-partition (16,384 per SMSP, warps dealt round-robin), so co-residency is decided per SMSP:
// shrink 8 warps (2 per SMSP) x <= 88 registers + expand 12 warps (3 per SMSP) x <= 104 registers
// = 15,104 <= 16,384, while two expand CTAs (19,968) never fit one SM; two shrink CTAs are kept
// apart by their SMEM (the launcher sizes a shrink CTA above half the SM's shared memory).
// The shrink has no producer warp: warp 0 refills a stage right after the tile's reduction
// barrier, which every warp passes only once it has read the stage.
template <int W>
__global__ void __maxnreg__(88)
    lora_shrink_ring_kernel(const __grid_constant__ RingArgs a, const __grid_constant__ MetaBlob<W> blob) {
    constexpr int ES = 2;
    extern __shared__ __align__(128) char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    float* part = reinterpret_cast<float*>(smem + kSPartOff);
    char* ring = smem + kSRingOff;
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ns = a.ns, stage_bytes = a.s_stage;
    unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 64 : nullptr;
    if (tr && tid == 0) tr[0] = gtime();
    if (W == 1) pdl_wait_cta();   // metadata uploaded by the preceding kernel
    const int32_t* offs = M + a.list_off;
    const int t0 = offs[blockIdx.x], nt = offs[blockIdx.x + 1] - t0;
    const int32_t* tiles = offs + a.n_cta + 1 + t0;
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_launch_dependents();
    // A rank rows of tile i -> stage i % ns (immutable pool pages: may precede the wait); x rows of
    // the tile's tokens into the same stage (lane 0, only after griddepcontrol.wait).  One full
    // barrier per stage use counts both (expect_tx covers A + x).  Warp 0 only.
    const uint64_t pol = policy_evict_first(), pol_x = policy_evict_normal();
    auto issue_a = [&](int i) {
        const int s = i % ns;
        const int w = tiles[i], gc = tw_gc(w), ks = tw_a(w), jb = tw_jb(w);
        const int r = gcf(M, gc, GC_RANK), poff = gcf(M, gc, GC_PAGE_OFF), ntok = gcf(M, gc, GC_NTOK);
        const DecodeJob& J = a.jobs[gcf(M, gc, GC_JOB)];
        const int j0 = jb * kShrinkRowsMma, nj = min(kShrinkRowsMma, r - j0);
        const int k0 = ks * kKSlice, nk = min(kKSlice, J.H_in - k0);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)((nj + ntok) * nk * ES));
        __syncwarp();
        if (lane < nj)
            bulk_g2s(ring + s * stage_bytes + lane * kSPitch,
                     J.A + ((size_t)pg_at(M, poff, j0 + lane) * J.H_in + k0) * ES, (uint32_t)(nk * ES), &full[s], pol);
    };
    auto issue_x = [&](int i) {
        const int s = i % ns;
        const int w = tiles[i], gc = tw_gc(w), ks = tw_a(w);
        const int ntok = gcf(M, gc, GC_NTOK), toff = gcf(M, gc, GC_TOK_OFF);
        const DecodeJob& J = a.jobs[gcf(M, gc, GC_JOB)];
        const int k0 = ks * kKSlice, nk = min(kKSlice, J.H_in - k0);
        for (int t = 0; t < ntok; ++t)
            bulk_g2s(ring + s * stage_bytes + (kShrinkRowsMma + t) * kSPitch,
                     J.x + ((size_t)M[toff + t] * J.x_ld + k0) * ES, (uint32_t)(nk * ES), &full[s], pol_x);
    };
    const int pre = min(ns, nt);
    if (warp == 0) {
        for (int i = 0; i < pre; ++i) issue_a(i);
        // x, and the v scratch overwritten below, may belong to the preceding kernel in the stream
        if (lane == 0) {
            pdl_wait();
            for (int i = 0; i < pre; ++i) issue_x(i);
        }
        __syncwarp();
    }
    consumer_sync();
    if (tr && tid == 0) tr[1] = gtime();
    const int g = lane >> 2, c = lane & 3;
    for (int i = 0; i < nt; ++i) {
        const int w = tiles[i], gc = tw_gc(w), ks = tw_a(w), jb = tw_jb(w);
        const int r = gcf(M, gc, GC_RANK), ntok = gcf(M, gc, GC_NTOK);
        const DecodeJob& J = a.jobs[gcf(M, gc, GC_JOB)];
        const int j0 = jb * kShrinkRowsMma, nj = min(kShrinkRowsMma, r - j0);
        const int nk = min(kKSlice, J.H_in - ks * kKSlice);
        const int s = i % ns;
        mbar_wait(&full[s], (i / ns) & 1);
        const char* st = ring + s * stage_bytes;
        uint4 ra[4], rb[4], xr[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int k = warp * 128 + b * 32 + c * 8;
            const bool kin = k < nk;
            ra[b] = (g < nj && kin) ? lds128(st + g * kSPitch + k * ES) : make_uint4(0u, 0u, 0u, 0u);
            rb[b] = (g + 8 < nj && kin) ? lds128(st + (g + 8) * kSPitch + k * ES) : make_uint4(0u, 0u, 0u, 0u);
            xr[b] = (g < ntok && kin) ? lds128(st + (kShrinkRowsMma + g) * kSPitch + k * ES) : make_uint4(0u, 0u, 0u, 0u);
        }
        float acc[4][4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            acc[b][0] = acc[b][1] = acc[b][2] = acc[b][3] = 0.f;
            mma_bf16(acc[b], ra[b].x, rb[b].x, ra[b].y, rb[b].y, xr[b].x, xr[b].y);
            mma_bf16(acc[b], ra[b].z, rb[b].z, ra[b].w, rb[b].w, xr[b].z, xr[b].w);
        }
        float* pw = part + ((i & 1) * kRingWarps + warp) * (16 * 8);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // fixed-order pairwise sum of the warp's 4 k-blocks (same order as the PDL pair)
            const float v = (acc[0][q] + acc[1][q]) + (acc[2][q] + acc[3][q]);
            pw[(g + ((q & 2) ? 8 : 0)) * 8 + 2 * c + (q & 1)] = v;
        }
        consumer_sync();   // every warp has read stage s and written its partial
        if (warp == 0 && i + ns < nt) {
            issue_a(i + ns);
            if (lane == 0) issue_x(i + ns);
            __syncwarp();
        }
        const int padr = j0 + nj == r ? v_stride(r) - r : 0;   // zero tail of the row stride
        if (tid < (nj + padr) * ntok) {
            const int row = tid / ntok, t = tid - row * ntok;
            float v = 0.f;
            if (row < nj) {
                const float* pp = part + (i & 1) * kRingWarps * 128 + row * 8 + t;
#pragma unroll
                for (int q = 0; q < kRingWarps; ++q) v += pp[q * 128];
            }
            a.vbuf[gcf(M, gc, GC_VOFF) + (ks * ntok + t) * v_stride(r) + j0 + row] = v;
        }
        if (tr && tid == 0 && i < 60) tr[2 + i] = gtime();
    }
    if (tr && tid == 0) { tr[62] = smid(); tr[63] = gtime(); }
}

// ------------------------------------------------------------------ expand
// warps 0-7 consumers, warp 8 B producer, warp 9 loader (y rows + v of the next units, after the
// wait), warps 10-11 idle (they exit at once: their registers keep a second expand CTA off the SM)
template <int W>
__global__ void __maxnreg__(104)
    lora_expand_ring_kernel(const __grid_constant__ RingArgs a, const __grid_constant__ MetaBlob<W> blob) {
    constexpr int ES = 2;
    extern __shared__ __align__(128) char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 8;
    uint64_t* ybar = full + 16;                    // [2] y rows of unit buffer b landed (tx)
    uint64_t* vfull = full + 18;                   // [2] v of unit buffer b staged (loader arrive)
    uint64_t* ufree = full + 20;                   // [2] unit buffer b free again (8 consumer warps)
    char* zero = smem + 192;                       // 64 zero bytes
    const int vpitch = a.e_vpitch;
    char* vbase = smem + a.e_voff;                 // [2 units][hi, lo][8 tokens][vpitch] bf16
    char* ybase = smem + a.e_yoff;                 // [2 units][max tokens][kEPitch]
    char* ring = smem + a.e_ringoff;
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ns = a.ns;
    unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 64 : nullptr;
    if (tr && tid == 0) tr[0] = gtime();
    if (W == 1) pdl_wait_cta();
    const int32_t* offs = M + a.list_off;
    const int t0 = offs[blockIdx.x], nt = offs[blockIdx.x + 1] - t0;
    const int32_t* tiles = offs + a.n_cta + 1 + t0;
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kRingWarps);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&ybar[b], 1);
            mbar_init(&vfull[b], 1);
            mbar_init(&ufree[b], kRingWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 16) reinterpret_cast<uint32_t*>(zero)[tid] = 0u;
    __syncthreads();
    pdl_launch_dependents();

    if (warp >= kRingWarps + 2) return;
    if (warp == kRingWarps) {
        // producer: B rows of every tile (16 rank rows x <= 1024 columns), HBM -> ring
        const uint64_t pol = policy_evict_first();
        for (int i = 0; i < nt; ++i) {
            const int s = i % ns;
            if (i >= ns) mbar_wait(&empty[s], ((i / ns) + 1) & 1);
            const int w = tiles[i], gc = tw_gc(w), cs = tw_a(w), jb = tw_jb(w);
            const int r = gcf(M, gc, GC_RANK), poff = gcf(M, gc, GC_PAGE_OFF);
            const DecodeJob& J = a.jobs[gcf(M, gc, GC_JOB)];
            const int j0 = jb * 16, nj = min(16, r - j0);
            const int n0 = cs * kECols, nc = min(kECols, J.H_out - n0);
            if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(nj * nc * ES));
            __syncwarp();
            if (lane < nj)
                bulk_g2s(ring + s * kEStage + lane * kEPitch,
                         J.B + ((size_t)pg_at(M, poff, j0 + lane) * J.H_out + n0) * ES, (uint32_t)(nc * ES), &full[s], pol);
            if (tw_first(w)) {
                const int ntok = gcf(M, gc, GC_NTOK);
                if (lane < ntok)
                    prefetch_l2(J.y + ((size_t)M[gcf(M, gc, GC_TOK_OFF) + lane] * J.y_ld + n0) * ES, (uint32_t)(nc * ES));
            }
        }
        return;
    }
    if (warp == kRingWarps + 1) {
        // loader: per unit (in list order, two buffers ahead of the consumers), after the wait:
        // y rows -> ybuf (bulk copies, tx barrier), v = s · Σ_ks partials (slice order) -> bf16 hi + lo
        if (lane == 0) pdl_wait();   // v from the shrink kernel, y from whoever wrote it
        __syncwarp();
        int u = 0;
        for (int i = 0; i < nt; ++i) {
            const int w = tiles[i];
            if (!tw_first(w)) continue;
            const int ub = u & 1;
            if (u >= 2) mbar_wait(&ufree[ub], ((u >> 1) + 1) & 1);
            const int gc = tw_gc(w);
            const int r = gcf(M, gc, GC_RANK), ntok = gcf(M, gc, GC_NTOK), toff = gcf(M, gc, GC_TOK_OFF);
            const DecodeJob& J = a.jobs[gcf(M, gc, GC_JOB)];
            const int n0 = tw_a(w) * kECols, nc = min(kECols, J.H_out - n0);
            char* yb = ybase + ub * a.e_ybuf;
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // ybuf last read by generic loads
                mbar_arrive_expect_tx(&ybar[ub], (uint32_t)(ntok * nc * ES));
                for (int t = 0; t < ntok; ++t)
                    bulk_g2s(yb + t * kEPitch, J.y + ((size_t)M[toff + t] * J.y_ld + n0) * ES, (uint32_t)(nc * ES),
                             &ybar[ub], policy_evict_normal());
            }
            const int rp = (r + 15) & ~15, vs = v_stride(r), ksplit = J.ksplit;
            const float* vsrc = a.vbuf + gcf(M, gc, GC_VOFF);
            const float scale = __int_as_float(gcf(M, gc, GC_SCALE));
            char* vhi = vbase + ub * (2 * kTokChunkMma * vpitch);
            char* vlo = vhi + kTokChunkMma * vpitch;
            const int n4 = ntok * (rp / 4);   // float4 groups of 4 ranks
            for (int e = lane; e < n4; e += 32) {
                const int t = e / (rp / 4), j = (e - t * (rp / 4)) * 4;
                float v[4] = {0.f, 0.f, 0.f, 0.f};
                if (j < vs) {   // v_stride(r) is a multiple of 4: the whole float4 is inside the row
                    const float* src = vsrc + t * vs + j;
                    const int stride = ntok * vs;
                    for (int k0 = 0; k0 < ksplit; k0 += 4) {
                        float4 p[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            p[q] = k0 + q < ksplit ? ldg_cg_f4(src + (k0 + q) * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            v[0] += p[q].x;
                            v[1] += p[q].y;
                            v[2] += p[q].z;
                            v[3] += p[q].w;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float vv = j + q < r ? v[q] * scale : 0.f;
                    const __nv_bfloat16 hi = __float2bfloat16_rn(vv);
                    const __nv_bfloat16 lo = __float2bfloat16_rn(vv - __bfloat162float(hi));
                    *reinterpret_cast<__nv_bfloat16*>(vhi + t * vpitch + (j + q) * 2) = hi;
                    *reinterpret_cast<__nv_bfloat16*>(vlo + t * vpitch + (j + q) * 2) = lo;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&vfull[ub]);
            ++u;
        }
        return;
    }

    if (tid == 0) pdl_wait();   // (y is written below; its producers must be complete)
    consumer_sync();
    if (tr && tid == 0) tr[1] = gtime();
    // mma operand lanes (as the PDL pair): B^T via ldmatrix.x4.trans, v via ldmatrix.x2
    const int am = lane >> 3, ai = lane & 7;
    const int aj = ai + ((am & 2) ? 8 : 0), an = (am & 1) * 8;
    const int vt = lane & 7, vh = (lane >> 3) & 1;
    const int g = lane >> 2, cc = lane & 3;
    const uint32_t zaddr = smem_u32(zero);
    const int colw = warp * 128;   // this warp's 128 columns of the unit's slice
    float d[8][4];
    int u = 0, ub = 0;
    int ntok = 0, nc = 0, n0 = 0, toff = 0, r = 0;
    const DecodeJob* Jp = &a.jobs[0];
    for (int i = 0; i < nt; ++i) {
        const int w = tiles[i], gc = tw_gc(w), jb = tw_jb(w);
        if (tw_first(w)) {
            ub = u & 1;
            r = gcf(M, gc, GC_RANK);
            ntok = gcf(M, gc, GC_NTOK);
            toff = gcf(M, gc, GC_TOK_OFF);
            Jp = &a.jobs[gcf(M, gc, GC_JOB)];
            n0 = tw_a(w) * kECols;
            nc = min(kECols, Jp->H_out - n0);
#pragma unroll
            for (int m = 0; m < 8; ++m) d[m][0] = d[m][1] = d[m][2] = d[m][3] = 0.f;
            mbar_wait(&vfull[ub], (u >> 1) & 1);
        }
        const int s = i % ns;
        mbar_wait(&full[s], (i / ns) & 1);
        {
            const int nj = min(16, r - jb * 16);
            const uint32_t st = smem_u32(ring + s * kEStage);
            const uint32_t vhb = smem_u32(vbase + ub * (2 * kTokChunkMma * vpitch)) + vt * vpitch + vh * 16 + jb * 32;
            const uint32_t vlb = vhb + kTokChunkMma * vpitch;
            uint32_t h0, h1, l0, l1;
            ldsm_x2(h0, h1, vhb);
            ldsm_x2(l0, l1, vlb);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int col16 = colw + m * 16;
                if (col16 < nc) {
                    uint32_t f0, f1, f2, f3;
                    ldsm_x4_trans(f0, f1, f2, f3, aj < nj ? st + aj * kEPitch + (col16 + an) * ES : zaddr);
                    mma_bf16(d[m], f0, f1, f2, f3, h0, h1);
                    mma_bf16(d[m], f0, f1, f2, f3, l0, l1);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (tw_last(w)) {
            char* yb = ybase + ub * a.e_ybuf;
            mbar_wait(&ybar[ub], (u >> 1) & 1);
            // D (fp32, [column g | g+8][tokens 2cc, 2cc+1]) added into the staged y, one rounding
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int col16 = colw + m * 16;
                if (col16 < nc) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int col = col16 + g + ((q & 2) ? 8 : 0), t = 2 * cc + (q & 1);
                        if (t < ntok && col < nc) {
                            __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(yb + t * kEPitch + col * ES);
                            *p = __float2bfloat16_rn(__bfloat162float(*p) + d[m][q]);
                        }
                    }
                }
            }
            consumer_sync();
            const int vpr = nc / 8;
            for (int e = tid; e < ntok * vpr; e += kRingConsumers) {
                const int t = e / vpr, q = e - t * vpr;
                stg128_na(Jp->y + ((size_t)M[toff + t] * Jp->y_ld + n0 + q * 8) * ES, lds128(yb + t * kEPitch + q * 16));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ufree[ub]);   // this warp is done with the unit's v and y buffers
            ++u;
        }
        if (tr && tid == 0 && i < 60) tr[2 + i] = gtime();
    }
    if (tr && tid == 0) { tr[62] = smid(); tr[63] = gtime(); }
}

// ------------------------------------------------------------------ host launcher
template <typename K, typename... Args>
static cudaError_t launch_pdl_ring(K kernel, int grid, int block, int smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Longest-processing-time-first assignment of weighted items to n bins (ties: lowest bin), each
// bin's items in assignment order.  out_off[n + 1], out_items = item indices.
static void lpt_assign(const std::vector<int64_t>& weight, int n, std::vector<int32_t>& out_off,
                       std::vector<int32_t>& out_items) {
    const int m = (int)weight.size();
    std::vector<int32_t> order(m);
    for (int i = 0; i < m; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return weight[x] > weight[y]; });
    std::vector<std::pair<int64_t, int32_t>> heap;   // (load, bin), min-heap
    heap.reserve(n);
    for (int b = 0; b < n; ++b) heap.push_back({0, b});
    auto cmp = [](const std::pair<int64_t, int32_t>& x, const std::pair<int64_t, int32_t>& y) {
        return x.first != y.first ? x.first > y.first : x.second > y.second;
    };
    std::make_heap(heap.begin(), heap.end(), cmp);
    std::vector<int32_t> bin_of(m);
    std::vector<int32_t> count(n, 0);
    for (int i : order) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto& top = heap.back();
        bin_of[i] = top.second;
        count[top.second] += 1;
        top.first += weight[i];
        std::push_heap(heap.begin(), heap.end(), cmp);
    }
    out_off.assign(n + 1, 0);
    for (int b = 0; b < n; ++b) out_off[b + 1] = out_off[b] + count[b];
    out_items.assign(m, 0);
    std::vector<int32_t> fill(out_off.begin(), out_off.end() - 1);
    for (int i : order) out_items[fill[bin_of[i]]++] = i;
}

template <int W>
static cudaError_t launch_ring_w(const RingArgs& as, const RingArgs& ae, int gs, int ge, int smem_s, int smem_e,
                                 const std::vector<int32_t>& words, cudaStream_t st, int* launches, int phases) {
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? 1ull << dev : 0;
    if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
        // the opt-in maximum, and the largest SMEM carveout: the driver otherwise configures an SM's
        // L1/SMEM split for the first kernel's one CTA, and the other kernel's CTA no longer fits beside it
        cudaError_t e = cudaFuncSetAttribute(lora_shrink_ring_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lora_expand_ring_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lora_shrink_ring_kernel<W>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lora_expand_ring_kernel<W>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    MetaBlob<W> blob;
    if (W > 1) {
        const int n = (int)words.size();
        for (int i = 0; i < n; ++i) blob.w[i] = words[i];
    }
    cudaError_t e = cudaSuccess;
    if ((phases & 1) && gs > 0) {
        e = launch_pdl_ring(lora_shrink_ring_kernel<W>, gs, kRingThreads, smem_s, st, as, blob);
        if (e != cudaSuccess) return e;
        *launches += 1;
    }
    if ((phases & 2) && ge > 0) {
        e = launch_pdl_ring(lora_expand_ring_kernel<W>, ge, kRingEThreads, smem_e, st, ae, blob);
        if (e != cudaSuccess) return e;
        *launches += 1;
    }
    return e;
}

// launches the ring pair for a bf16 plan (phases 3: full apply).  ring_cfg: 1 = default stage
// counts, else 0x100 | ns_shrink << 4 | ns_expand (experiments).  Returns a cudaError_t.
int launch_decode_ring(const Plan& pl, const DecodeLaunch& L, cudaStream_t st, int* launches, int ring_cfg) {
    RingArgs a;
    memset(&a, 0, sizeof(a));
    for (int j = 0; j < L.n_jobs && j < kMaxJobs; ++j) {
        const void* x = j == 0 ? L.x : L.more[j - 1].x;
        void* y = j == 0 ? L.y : L.more[j - 1].y;
        const void* A = j == 0 ? L.poolA : L.more[j - 1].poolA;
        const void* B = j == 0 ? L.poolB : L.more[j - 1].poolB;
        const int hin = j == 0 ? L.H_in : L.more[j - 1].H_in, hout = j == 0 ? L.H_out : L.more[j - 1].H_out;
        const int xld = j == 0 && L.x_ld > 0 ? (int)L.x_ld : hin, yld = j == 0 && L.y_ld > 0 ? (int)L.y_ld : hout;
        a.jobs[j] = DecodeJob{static_cast<const char*>(x), static_cast<char*>(y), static_cast<const char*>(A),
                              static_cast<const char*>(B), hin, hout, ksplit_of(hin, 2), xld, yld};
    }
    a.vbuf = L.vbuf;
    a.meta_global = L.meta_dev;
    // work lists: shrink tiles and expand units from the gc records
    const int32_t* gcr = pl.blob.data() + kHdrWords;
    static thread_local std::vector<int32_t> s_words, e_units_first, e_units_n;
    static thread_local std::vector<int64_t> s_w, e_w;
    s_words.clear(); s_w.clear(); e_units_first.clear(); e_units_n.clear(); e_w.clear();
    static thread_local std::vector<int32_t> e_words;
    e_words.clear();
    int maxr = 1, maxtok = 1;
    if (pl.n_gc >= (1 << 15) || pl.n_gc == 0) return -1;
    for (int gc = 0; gc < pl.n_gc; ++gc) {
        const int32_t* e = gcr + gc * kGcFields;
        const int r = e[GC_RANK], ntok = e[GC_NTOK];
        const DecodeJob& J = a.jobs[e[GC_JOB]];
        maxr = std::max(maxr, r);
        maxtok = std::max(maxtok, ntok);
        const int njb = (r + 15) / 16, ks_n = (J.H_in + kKSlice - 1) / kKSlice, cs_n = (J.H_out + kECols - 1) / kECols;
        if (njb > 16 || ks_n > 32 || cs_n > 32) return -1;   // tile-word fields
        for (int ks = 0; ks < ks_n; ++ks)
            for (int jb = 0; jb < njb; ++jb) {
                s_words.push_back(gc | ks << 15 | jb << 20);
                s_w.push_back((int64_t)std::min(16, r - jb * 16) * std::min(kKSlice, J.H_in - ks * kKSlice));
            }
        for (int cs = 0; cs < cs_n; ++cs) {
            e_units_first.push_back((int32_t)e_words.size());
            e_units_n.push_back(njb);
            e_w.push_back((int64_t)r * std::min(kECols, J.H_out - cs * kECols) + 2048);   // + per-unit v/y cost
            for (int jb = 0; jb < njb; ++jb)
                e_words.push_back(gc | cs << 15 | jb << 20 | (jb == 0 ? 1 << 24 : 0) | (jb == njb - 1 ? 1 << 25 : 0));
        }
    }
    const int gs = std::min<int>(L.num_sms, (int)s_words.size());
    const int ge = std::min<int>(L.num_sms, (int)e_units_first.size());
    static thread_local std::vector<int32_t> words, off, items;
    words.assign(pl.blob.begin(), pl.blob.begin() + pl.unit_tab);   // gc records, pages, tokens
    a.list_off = (int)words.size();
    RingArgs ae = a;
    lpt_assign(s_w, gs, off, items);
    words.insert(words.end(), off.begin(), off.end());
    for (int it : items) words.push_back(s_words[it]);
    ae.list_off = (int)words.size();
    lpt_assign(e_w, ge, off, items);
    words.insert(words.end(), off.begin(), off.end());
    {
        // expand list: unit offsets -> tile offsets
        std::vector<int32_t> toff(ge + 1, 0);
        for (int b = 0; b < ge; ++b) {
            int n = 0;
            for (int k = off[b]; k < off[b + 1]; ++k) n += e_units_n[items[k]];
            toff[b + 1] = toff[b] + n;
        }
        std::copy(toff.begin(), toff.end(), words.end() - (ge + 1));
        for (int it : items)
            for (int k = 0; k < e_units_n[it]; ++k) words.push_back(e_words[e_units_first[it] + k]);
    }
    a.n_cta = gs;
    ae.n_cta = ge;
    // smem layout and stage counts: one shrink CTA + one expand CTA per SM
    const int rp = (maxr + 15) & ~15;
    ae.e_vpitch = (rp + 8) * 2;
    ae.e_voff = 256;
    ae.e_yoff = (ae.e_voff + 2 * 2 * kTokChunkMma * ae.e_vpitch + 127) & ~127;
    ae.e_ybuf = maxtok * kEPitch;
    ae.e_ringoff = (ae.e_yoff + 2 * ae.e_ybuf + 127) & ~127;
    // stage counts.  Placement contract: one shrink CTA + one expand CTA per SM, never two of the
    // same kernel (two expand CTAs exceed the register file; a shrink CTA is padded above half the
    // SM's shared memory), so S + E + 2 KB reserved <= 228 KB with S >= kSMinSmem.
    a.s_stage = (kShrinkRowsMma + maxtok) * kSPitch;
    auto smem_s_of = [&](int ns) { return std::max(kSRingOff + ns * a.s_stage, kSMinSmem); };
    auto smem_e_of = [&](int ns) { return ae.e_ringoff + ns * kEStage; };
    auto fits = [&](int s_, int e_) {
        return smem_s_of(s_) + smem_e_of(e_) + 2 * kSmemReserved <= kSmemPerSM && smem_s_of(s_) <= 227 * 1024 &&
               smem_e_of(e_) <= 227 * 1024;
    };
    int ns_s = 0, ns_e = 0;
    if (ring_cfg & 0x100) {
        ns_s = std::max(1, std::min(kRingMaxStages, (ring_cfg >> 4) & 0xf));
        ns_e = std::max(1, std::min(kRingMaxStages, ring_cfg & 0xf));
        if (!fits(ns_s, ns_e)) return -1;
    } else {
        // the most stages in total, then the most expand stages (its B streams while the shrink computes)
        int best = -1;
        for (int e_ = 1; e_ <= kRingMaxStages; ++e_)
            for (int s_ = 1; s_ <= kRingMaxStages; ++s_)
                if (fits(s_, e_) && (s_ + e_) * 64 + e_ > best) { best = (s_ + e_) * 64 + e_; ns_s = s_; ns_e = e_; }
        if (best < 0 || ns_s + ns_e < 4) return -1;   // too little ring for this batch: the PDL pair
    }
    a.ns = ns_s;
    ae.ns = ns_e;
    const int smem_s = smem_s_of(ns_s);
    const int smem_e = smem_e_of(ns_e);
    a.trace = L.trace;
    ae.trace = L.trace ? L.trace + (size_t)L.num_sms * 64 : nullptr;
    const int n = (int)words.size();
    const int phases = L.phases;
    if (n <= 1024) return (int)launch_ring_w<1024>(a, ae, gs, ge, smem_s, smem_e, words, st, launches, phases);
    if (n <= 2048) return (int)launch_ring_w<2048>(a, ae, gs, ge, smem_s, smem_e, words, st, launches, phases);
    if (n <= 4096) return (int)launch_ring_w<4096>(a, ae, gs, ge, smem_s, smem_e, words, st, launches, phases);
    if (n <= kMaxParamBlobWords) return (int)launch_ring_w<kMaxParamBlobWords>(a, ae, gs, ge, smem_s, smem_e, words, st, launches, phases);
    return -1;   // too large for the kernel parameters: the PDL pair (device-memory metadata) takes it
}

}  // namespace lora
