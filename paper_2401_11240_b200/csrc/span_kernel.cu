// span_kernel.cu -- N1c: the bf16 decode delta as ONE grid per apply, sm_100a.
//
// Computes, per (adapter group-chunk gc of <= 8 tokens, token t of gc):   (§2.1 Eq. 1)
//     v_t[j]  = s_g · Σ_k x_t[k] · A_g[k][j]       shrink, fp32 accumulation
//     y_t[n] += Σ_j v_t[j] · B_g[j][n]             expand, fp32 accumulation, one rounding
// with no padding to the batch's max rank (MBGMV semantics).
//
// Why one grid (DESIGN.md §6 N1c).  A decode apply moves ~17 MB (c2), 2.6 µs of HBM time, but
// a shrink grid -> expand grid chain spends ~5 µs in dependency latency: two grid completions,
// the v round trip through L2 and the x/y loads after each wait.  Here every gc is owned by a
// *span* of s CTAs inside one thread-block cluster (s ∝ rank, a power of two <= the cluster
// size, so every CTA moves about the same adapter bytes).  CTA i of the span owns slice i of
// H_in (its part of the shrink) and slice i of H_out (its part of the expand):
//   1. before griddepcontrol.wait it streams its A and B rank rows (immutable pool pages) into
//      a ring of smem stages with 16-B cp.async (LDGSTS; one mbarrier per stage), so the whole
//      apply's adapter bytes are in flight while the preceding kernel in the stream finishes;
//   2. after the wait it bulk-copies its x rows and y rows (cp.async.bulk, mbarrier tx count);
//   3. shrink: bf16 mma.sync (m16n8k16, fp32 accumulate) of its A slice against x, reduced over
//      warps in a fixed order into a partial v [r][8] in its own smem;
//   4. cluster barrier; every CTA of the span sums the s partials over distributed shared memory
//      (ld.shared::cluster, fixed order q = 0..s-1), scales, splits v into bf16 hi + lo;
//   5. expand: swap-AB MMAs D[col][tok] = B^T · v^T over its B slice, added into the staged y
//      rows with one rounding, written back with 16-B stores.
// No global scratch, no atomics, no spin waits: the result of a token is a fixed function of
// (x_t, adapter) because the span and all reduction orders depend only on (r, H_in, H_out).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

struct SpanJob {
    const char* x;
    char* y;
    const char* tmaps;   // device array of kSpanMaps CUtensorMaps: A boxes {64, 8 << i}, then B boxes
    int H_in, H_out;
};

struct SpanArgs {
    SpanJob jobs[kMaxJobs];
    unsigned long long* trace;   // debug: 16 timestamps per CTA, or null
    int stage_bytes, n_stages;
    // dynamic smem layout (bytes), sized per launch from the batch's largest rank / slices
    int vp_off, v_off, v_pitch, x_off, x_pitch, y_off, y_pitch, ring_off, smem;
};

template <int W>
struct SpanBlob {
    int32_t w[W];
};

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "SPAN_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra SPAN_WAIT;\n}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// D[16x8] += A[16x16] (row) * B[16x8] (col), bf16 inputs, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void st_global_v4(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// 2D TMA box load (tensor map in global memory): box at element coordinates {c0 = column, c1 = page}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// Ring stage layout of a chunk of rows8 rows (rank rounded up to 8) x W columns, as the TMA boxes
// {64 columns, 8..128 rows} with the 128-B swizzle leave it: column block b = W/64 blocks of
// [rows8][128 B]; 16-B piece q of row j sits at block q/8, row j, position (q%8) ^ (j%8)
// (every ldmatrix of 8 rows hits 8 distinct bank groups).  Stage and block bases are 1024-B aligned.
__device__ __forceinline__ uint32_t chunk_addr(uint32_t stage, int rows8, int row, int q) {
    return stage + (q >> 3) * rows8 * 128 + row * 128 + (((q & 7) ^ (row & 7)) << 4);
}

struct Rec {
    int job, s, ci, leader, r, ntok, pg, tk, kc, nc, k0, nk, n0, nn;
    float scale;
};

__device__ __forceinline__ Rec decode_rec(const int32_t* w) {
    Rec d;
    const uint32_t w0 = (uint32_t)w[0], w1 = (uint32_t)w[1], w5 = (uint32_t)w[5], w6 = (uint32_t)w[6],
                   w7 = (uint32_t)w[7];
    d.job = w0 & 15;
    d.s = (w0 >> 4) & 255;
    d.ci = (w0 >> 12) & 255;
    d.leader = (w0 >> 20) & 255;
    d.r = w1 & 0xffff;
    d.ntok = w1 >> 16;
    d.pg = w[2];
    d.tk = w[3];
    d.scale = __int_as_float(w[4]);
    d.kc = w5 & 0xffff;
    d.nc = w5 >> 16;
    d.k0 = w6 & 0xffff;
    d.nk = w6 >> 16;
    d.n0 = w7 & 0xffff;
    d.nn = w7 >> 16;
    return d;
}

}  // namespace

// smem: [0, 8*kSpanMaxStages) stage barriers | [96] x/y barrier | [128, 160) tokens | [160, 224)
// zero bytes | vpart fp32 [rp][8] | warp partials (aliased by
// v hi/lo bf16 [8][v_pitch] x 2) | x rows [8][x_pitch] | y rows [8][y_pitch] | ring stages
template <int W>
__global__ void __launch_bounds__(kConsumerThreads, 2)
    lora_span_kernel(const __grid_constant__ SpanArgs a, const __grid_constant__ SpanBlob<W> blob) {
    extern __shared__ __align__(1024) char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint64_t* bar_xy = bars + kSpanMaxStages;
    int* stok = reinterpret_cast<int*>(smem + 128);
    char* zero = smem + 160;
    float* vpart = reinterpret_cast<float*>(smem + a.vp_off);
    float* wpart = reinterpret_cast<float*>(smem + a.v_off);
    char* xs = smem + a.x_off;
    char* ys = smem + a.y_off;
    const uint32_t ring = su32(smem + a.ring_off);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NS = a.n_stages, SB = a.stage_bytes;
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 1] = gtime();

    const Rec d = decode_rec(blob.w + kSpanRecWords * blockIdx.x);
    const SpanJob J = a.jobs[d.job];
    const int r = d.r;
    const int nA = d.nk > 0 ? (d.nk + d.kc - 1) / d.kc : 0;
    const int nB = d.nn > 0 ? (d.nn + d.nc - 1) / d.nc : 0;
    const int NC = r > 0 ? nA + nB : 0;

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
        mbar_init(bar_xy, kConsumerThreads);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 14] = gtime();
    if (tid < 16) reinterpret_cast<uint32_t*>(zero)[tid] = 0u;
    if (tid < kSpanTok) stok[tid] = tid < d.ntok ? blob.w[d.tk + tid] : -1;
    // a ragged last k-slice (nk % 16 == 8) reads 8 x columns past nk in its last k-step: zero
    // them (the bulk copy below writes [0, nk) only), so 0-filled A columns never meet garbage
    if (tid < kSpanTok && (d.nk & 15)) *reinterpret_cast<uint4*>(xs + tid * a.x_pitch + d.nk * 2) = make_uint4(0, 0, 0, 0);
    __syncthreads();

    // ---- ring producer: chunk c (A chunks first, then B chunks) -> stage c % NS.  The gc's rank
    // rows are contiguous pages [pg, pg + r): a chunk is W/64 column blocks, each loaded as 2D TMA
    // boxes {64 columns, 8..128 rows} (one request moves up to 16 KB; per-request cost is what
    // limits small copies).  Rows r..rows8-1 of a box are neighbouring pages: loaded, never read.
    const int rows8 = (r + 7) & ~7;
    auto issue = [&](int c) {
        if (warp != 0 || lane != 0) return;
        const bool isA = c < nA;
        const int Wc = isA ? d.kc : d.nc;
        const int cb = isA ? c : c - nA;
        const int col0 = (isA ? d.k0 : d.n0) + cb * Wc;
        const int width = min(Wc, (isA ? d.nk : d.nn) - cb * Wc);
        const int nblk = (width + 63) >> 6;
        const char* maps = J.tmaps + (isA ? 0 : kSpanBoxKinds) * 128;
        const uint32_t stage = ring + (c % NS) * SB;
        mbar_expect_tx(&bars[c % NS], (uint32_t)(nblk * rows8 * 128));
        for (int b = 0; b < nblk; ++b) {
            int row = 0;
            for (int k = kSpanBoxKinds - 1; k >= 0; --k) {
                const int R = 8 << k;
                while (rows8 - row >= R) {
                    tma_load_2d(stage + b * rows8 * 128 + row * 128, maps + k * 128, col0 + b * 64, d.pg + row, &bars[c % NS]);
                    row += R;
                }
            }
        }
    };
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 15] = gtime();
    const int npre = NC < NS ? NC : NS;
    for (int c = 0; c < npre; ++c) issue(c);
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 7] = gtime();
    // warm L2 with this CTA's x / y rows (safe before the wait: L2 is the point of coherence)
    if (r > 0 && warp == 0 && lane < d.ntok) {
        const int t = stok[lane];
        if (d.nk > 0) prefetch_l2(J.x + ((size_t)t * J.H_in + d.k0) * 2, (uint32_t)d.nk * 2);
        if (d.nn > 0) prefetch_l2(J.y + ((size_t)t * J.H_out + d.n0) * 2, (uint32_t)d.nn * 2);
    }
    pdl_launch_dependents();

    const int RT = (r + 15) >> 4;   // 16-row rank tiles
    int WPT = 1, tile0 = warp, ntl = 0;
    if (RT > 0 && RT <= 8) {
        int rt2 = 1;
        while (rt2 < RT) rt2 <<= 1;
        WPT = 8 / rt2;
        tile0 = warp / WPT;
        ntl = tile0 < RT ? 1 : 0;
    } else if (RT > 8) {
        ntl = warp + 8 < RT ? 2 : 1;
    }
    const int wsub = warp % WPT;

    if (r > 0) {
        // ---- x and y rows of the gc's tokens (may be written by the preceding kernel)
        if (tid == 0) pdl_wait();
        __syncthreads();
        if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 2] = gtime();
        {   // 16-B LDGSTS from every thread (many small rows: the TMA per-request cost would dominate)
            const int xv = d.nk >> 3, yv = d.nn >> 3;
            for (int i = tid; i < d.ntok * (xv + yv); i += kConsumerThreads) {
                const int t = i / (xv + yv), q = i - t * (xv + yv);
                const int tok = stok[t];
                if (q < xv)
                    cp16(su32(xs + t * a.x_pitch + q * 16), J.x + ((size_t)tok * J.H_in + d.k0 + q * 8) * 2);
                else
                    cp16(su32(ys + t * a.y_pitch + (q - xv) * 16), J.y + ((size_t)tok * J.H_out + d.n0 + (q - xv) * 8) * 2);
            }
            cp_async_arrive(bar_xy);
        }
        // x rows of tokens >= ntok are never loaded: they only feed MMA columns that are dropped
        float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        // ldmatrix lane roles
        const int lr = lane & 7, lm = lane >> 3;
        const uint32_t zaddr = su32(zero);
        const uint32_t xbase = su32(xs) + lr * a.x_pitch;
        bool xy_ready = false;
        // ---- shrink over the A chunks
        for (int c = 0; c < nA; ++c) {
            mbar_wait(&bars[c % NS], (uint32_t)((c / NS) & 1));
            if (!xy_ready) {
                mbar_wait(bar_xy, 0);
                xy_ready = true;
                if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 3] = gtime();
            }
            if (a.trace && tid == 0 && c == nA - 1) a.trace[(size_t)blockIdx.x * 16 + 8] = gtime();
            const uint32_t stage = ring + (c % NS) * SB;
            const int Wc = d.kc;
            const int width = min(Wc, d.nk - c * Wc);
            const int nks = (width + 15) >> 4;
            const int gk0 = c * (Wc >> 4);   // global k-step of the chunk's first step
            for (int ks = 0; ks < nks; ++ks) {
                if (((gk0 + ks) % WPT) != wsub || ntl == 0) continue;
                uint32_t b0, b1;
                // x: token rows (lanes 0-7 k-piece 2ks, lanes 8-15 piece 2ks+1)
                ldsm_x2(b0, b1, xbase + ((gk0 + ks) * 16 + ((lm & 1) << 3)) * 2);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (q < ntl) {
                        const int tile = RT > 8 ? warp + 8 * q : tile0;
                        const int row = tile * 16 + lr + ((lm & 1) << 3);
                        const int piece = ks * 2 + (lm >> 1);
                        uint32_t af[4];
                        ldsm_x4(af, row < r ? chunk_addr(stage, rows8, row, piece) : zaddr);
                        mma16816(acc[q], af, b0, b1);
                    }
                }
            }
            __syncthreads();   // stage c is free
            if (c + NS < NC) issue(c + NS);
        }
        if (!xy_ready) {
            mbar_wait(bar_xy, 0);
            xy_ready = true;
        }
        // ---- warp partials -> CTA partial v [rp][8] (fixed order over the WPT warps of a tile)
        {
            const int g = lane >> 2, cc = lane & 3;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q < ntl) {
                    float* pw = wpart + (warp * 2 + q) * 128;
#pragma unroll
                    for (int e = 0; e < 4; ++e) pw[(g + ((e & 2) ? 8 : 0)) * 8 + 2 * cc + (e & 1)] = acc[q][e];
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < RT * 128; i += kConsumerThreads) {
            const int tile = i >> 7, e = i & 127;
            float v = 0.f;
            if (RT <= 8) {
                for (int w = 0; w < WPT; ++w) v += wpart[((tile * WPT + w) * 2) * 128 + e];
            } else {
                v = wpart[((tile & 7) * 2 + (tile >> 3)) * 128 + e];
            }
            vpart[tile * 128 + e] = v;
        }
    }
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 9] = gtime();
    // ---- span reduction over distributed shared memory
    cluster_arrive();
    cluster_wait();
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 6] = gtime();
    char* vhi = smem + a.v_off;   // reuses the warp-partial region (dead after the barrier)
    char* vlo = vhi + kSpanTok * a.v_pitch;
    if (r > 0) {
        const int rp = RT * 16;
        const uint32_t my = su32(vpart);
        for (int i = tid; i < rp * 8; i += kConsumerThreads) {
            const int j = i >> 3, t = i & 7;
            float v = 0.f;
            if (j < r) {
                float p[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    p[q] = q < d.s ? ld_dsmem(mapa(my + i * 4, (uint32_t)(d.leader + q))) : 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q) v += p[q];
                v *= d.scale;
            }
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
            *reinterpret_cast<__nv_bfloat16*>(vhi + t * a.v_pitch + j * 2) = h;
            *reinterpret_cast<__nv_bfloat16*>(vlo + t * a.v_pitch + j * 2) = l;
        }
    }
    if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 13] = gtime();
    cluster_arrive();   // done reading the peers' partials (waited for before exit)
    __syncthreads();
    if (r > 0) {
        // ---- expand over the B chunks: D[col][tok] = B^T[col][rank] · v^T[rank][tok]
        const int am = lane >> 3, ai = lane & 7;
        const int aj = ai + ((am & 2) ? 8 : 0), an = (am & 1) * 8;   // ldmatrix.trans roles
        const int vt = lane & 7, vh = (lane >> 3) & 1;
        const uint32_t vhi_b = su32(vhi) + vt * a.v_pitch + vh * 16;
        const uint32_t vlo_b = su32(vlo) + vt * a.v_pitch + vh * 16;
        const uint32_t zaddr = su32(zero);
        const int g = lane >> 2, cc = lane & 3;
        for (int c = nA; c < NC; ++c) {
            mbar_wait(&bars[c % NS], (uint32_t)((c / NS) & 1));
            if (a.trace && tid == 0 && c == nA) a.trace[(size_t)blockIdx.x * 16 + 10] = gtime();
            if (a.trace && tid == 0 && c == NC - 1) a.trace[(size_t)blockIdx.x * 16 + 11] = gtime();
            const uint32_t stage = ring + (c % NS) * SB;
            const int cb = c - nA, Wc = d.nc;
            const int width = min(Wc, d.nn - cb * Wc);
            const int ntiles = (width + 15) >> 4;
            for (int tile = warp; tile < ntiles; tile += kConsumerWarps) {
                float dd[4] = {0.f, 0.f, 0.f, 0.f};
                for (int rs = 0; rs < RT; ++rs) {
                    const int j = rs * 16 + aj;
                    uint32_t af[4], h0, h1, l0, l1;
                    ldsm_x4_trans(af, j < r ? chunk_addr(stage, rows8, j, tile * 2 + (an >> 3)) : zaddr);
                    ldsm_x2(h0, h1, vhi_b + rs * 32);
                    ldsm_x2(l0, l1, vlo_b + rs * 32);
                    mma16816(dd, af, h0, h1);
                    mma16816(dd, af, l0, l1);
                }
                // D: column g (+8), tokens 2cc, 2cc+1 -> y rows staged in smem, one rounding
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int t = 2 * cc + (e & 1);
                    const int n = cb * Wc + tile * 16 + g + ((e & 2) ? 8 : 0);
                    if (t < d.ntok && n < d.nn) {
                        __nv_bfloat16* py = reinterpret_cast<__nv_bfloat16*>(ys + t * a.y_pitch + n * 2);
                        *py = __float2bfloat16_rn(__bfloat162float(*py) + dd[e]);
                    }
                }
            }
            __syncthreads();   // stage c is free
            if (c + NS < NC) issue(c + NS);
        }
        if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * 16 + 12] = gtime();
        // ---- y rows back to HBM (16-B stores)
        const int vpr = d.nn >> 3;
        for (int i = tid; i < d.ntok * vpr; i += kConsumerThreads) {
            const int t = i / vpr, q = i - t * vpr;
            const uint4 v = *reinterpret_cast<const uint4*>(ys + t * a.y_pitch + q * 16);
            st_global_v4(J.y + ((size_t)stok[t] * J.H_out + d.n0 + q * 8) * 2, v);
        }
    }
    if (a.trace && tid == 0) {
        a.trace[(size_t)blockIdx.x * 16 + 0] = smid();
        a.trace[(size_t)blockIdx.x * 16 + 4] = r;
        a.trace[(size_t)blockIdx.x * 16 + 5] = gtime();
    }
    cluster_wait();   // peers no longer read this CTA's partial
}

// ------------------------------------------------------------------ host side
static SpanParams g_params;
static bool g_params_init = false;

const SpanParams& span_params() {
    if (!g_params_init) {
        // experiment knobs (sweeps); the defaults are the measured best (DESIGN.md §6 N1c)
        if (const char* e = getenv("LORA_SPAN_CLUSTER")) g_params.cluster = atoi(e);
        if (const char* e = getenv("LORA_SPAN_TARGET")) g_params.target_bytes = atoi(e);
        if (const char* e = getenv("LORA_SPAN_STAGE")) g_params.stage_bytes = atoi(e);
        if (const char* e = getenv("LORA_SPAN_STAGES")) g_params.n_stages = atoi(e);
        if (g_params.n_stages > kSpanMaxStages) g_params.n_stages = kSpanMaxStages;
        if (g_params.n_stages < 2) g_params.n_stages = 2;
        if (g_params.stage_bytes < 8192) g_params.stage_bytes = 8192;   // r = 256 rows x 16 columns
        if (g_params.cluster < 1 || g_params.cluster > 16 || (g_params.cluster & (g_params.cluster - 1))) g_params.cluster = 16;
        g_params_init = true;
    }
    return g_params;
}

static int span_layout(const Plan& pl, SpanArgs& a) {
    const SpanParams& sp = span_params();
    // a chunk is rows8 x W bf16 with W >= 64 (one TMA box column block): 1024-B aligned stages
    const int rows8 = (pl.span_max_rank + 7) & ~7;
    a.stage_bytes = sp.stage_bytes > rows8 * 128 ? sp.stage_bytes : rows8 * 128;
    a.stage_bytes = (a.stage_bytes + 1023) & ~1023;
    a.n_stages = sp.n_stages;
    const int rp = (pl.span_max_rank + 15) & ~15;
    int off = 256;
    a.vp_off = off;
    off += rp * 8 * 4;
    a.v_off = off;
    a.v_pitch = (rp + 8) * 2;
    const int wpart_bytes = kConsumerWarps * 2 * 128 * 4;
    const int v_bytes = 2 * kSpanTok * a.v_pitch;
    off += wpart_bytes > v_bytes ? wpart_bytes : v_bytes;
    off = (off + 127) & ~127;
    a.x_off = off;
    a.x_pitch = pl.span_max_sk * 2 + 16;
    off += kSpanTok * a.x_pitch;
    a.y_off = off;
    a.y_pitch = pl.span_max_sn * 2 + 16;
    off += kSpanTok * a.y_pitch;
    off = (off + 1023) & ~1023;
    a.ring_off = off;
    off += a.n_stages * a.stage_bytes;
    a.smem = off;
    return off;
}

bool span_fits(const Plan& pl) {
    if (pl.span_cluster == 0) return false;
    SpanArgs a;
    return span_layout(pl, a) <= 227 * 1024;
}

template <int W>
static cudaError_t launch_span_w(const Plan& pl, const SpanArgs& a, cudaStream_t st) {
    static bool configured[17] = {};
    const int cl = pl.span_cluster;
    if (!configured[cl]) {
        cudaError_t e = cudaFuncSetAttribute(lora_span_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e == cudaSuccess && cl > 8)
            e = cudaFuncSetAttribute(lora_span_kernel<W>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured[cl] = true;
    }
    SpanBlob<W> blob;
    const int n = (int)pl.span_blob.size();
    memcpy(blob.w, pl.span_blob.data(), (size_t)n * 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.n_span_cta);
    cfg.blockDim = dim3(kConsumerThreads);
    cfg.dynamicSmemBytes = a.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cl;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, lora_span_kernel<W>, a, blob);
}

constexpr int kSpanMaxBlobWords = 7936;

int make_tmap_bf16(void* tm_out, const void* base, int64_t rows, int64_t cols, int box_rows);   // prefill_kernel.cu

int span_make_tmaps(void* host_out, const void* dA, const void* dB, int n_rows, int H_in, int H_out) {
    char* o = static_cast<char*>(host_out);
    for (int k = 0; k < kSpanBoxKinds; ++k) {
        if (make_tmap_bf16(o + k * 128, dA, n_rows, H_in, 8 << k)) return 1;
        if (make_tmap_bf16(o + (kSpanBoxKinds + k) * 128, dB, n_rows, H_out, 8 << k)) return 1;
    }
    return 0;
}

int launch_span(const Plan& pl, const SpanLaunchDesc& L, cudaStream_t st, int* launches) {
    SpanArgs a;
    memset(&a, 0, sizeof(a));
    for (int j = 0; j < L.n_jobs && j < kMaxJobs; ++j)
        a.jobs[j] = SpanJob{static_cast<const char*>(L.x[j]), static_cast<char*>(L.y[j]),
                            static_cast<const char*>(L.tmaps[j]), L.H_in[j], L.H_out[j]};
    a.trace = L.trace;
    span_layout(pl, a);
    const int n = (int)pl.span_blob.size();
    cudaError_t e;
    if (n <= 2048)
        e = launch_span_w<2048>(pl, a, st);
    else if (n <= 4096)
        e = launch_span_w<4096>(pl, a, st);
    else if (n <= kSpanMaxBlobWords)
        e = launch_span_w<kSpanMaxBlobWords>(pl, a, st);
    else
        return (int)cudaErrorInvalidValue;
    if (e == cudaSuccess) *launches += 1;
    return (int)e;
}

int span_max_blob_words() { return kSpanMaxBlobWords; }

}  // namespace lora
