// decode_kernel.cu -- N1: the SIMT batched multi-adapter LoRA delta for decode tokens
// (and any token not routed to the tensor-core prefill kernel), sm_100a.
//
// Computes, per (adapter group g, token t of g):      (§2.1 Eq. 1)
//     v_t[j]  = s_g · Σ_k x_t[k] · A_g[k][j]          shrink, fp32 accumulation
//     y_t[n] += Σ_j v_t[j] · B_g[j][n]                expand, fp32 accumulation, one rounding
// with no padding to the batch's max rank (MBGMV semantics).
//
// Design (DESIGN.md §"N1"):
//  * Memory-bound on adapter bytes (the prior-art kernels already use > 70% of HBM
//    bandwidth).  Each CTA owns one work unit and streams its rank rows of A
//    (shrink) or B (expand) HBM -> SMEM with cp.async.bulk (the TMA bulk-copy engine,
//    SASS UBLKCP) issued by one warp, so a unit's whole 32 KB is in flight at once without
//    registers, and ~4 CTAs per SM keep >100 KB per SM in flight.
//  * Two kernels per apply, chained with programmatic dependent launch (PDL): every CTA
//    first issues the loads of its adapter rows (immutable pool pages), then signals
//    launch_dependents and only then executes griddepcontrol.wait before touching data a
//    preceding kernel may produce (x, y, the v scratch).  So the expand kernel's B rows
//    stream in while the shrink kernel runs, and the next apply's A rows while this apply
//    finishes -- the shrink -> expand dependency costs no global flags or atomics.
//  * v (the rank-r intermediate, fp32) goes through a small L2-resident scratch; partial
//    sums over k-slices and rank parts are reduced in a fixed order (no float atomics), so
//    a token's result is a fixed function of (x_t, adapter): bitwise reproducible and
//    independent of batch order (pin P6).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

struct DecodeJob {                // one pool's operands (lora_apply_multi fuses up to kMaxJobs)
    const char* x;
    char* y;
    const char* A;                // pool page arrays
    const char* B;
    int H_in, H_out, ksplit;
    int x_ld, y_ld;               // row strides of x and y in elements (H_in / H_out unless a TP shard view)
};

struct DecodeArgs {
    DecodeJob jobs[kMaxJobs];
    float* vbuf;
    const int32_t* meta_global;  // metadata in device memory (large batches) or null
    unsigned long long* trace;   // debug: per-unit timestamps, or null
    int n_shrink, n_expand, n_gc, n_jobs;
    int unit_tab;                // blob word offset of the per-unit table (plan.cpp append_unit_table)
    int unit_words;              // 3 (full unit records) or 1 (gc | local only: large batches)
    int e_smem;                  // bf16 expand: dynamic smem of the launch (the largest unit's layout)
    float* vred;                 // compact k-reduced v (TP split): written by the shrink kernel's last CTA of
                                 // each gc (tp_reduce_tail), read by the expand when v_compact is set
    int* gc_cnt;                 // TP shrink: per-gc arrival counters (zero between applies)
    int v_compact;
    int job_shrink_base[kMaxJobs];   // first unit of each fused job (units of a job are contiguous)
    int job_expand_base[kMaxJobs];
};

// job of unit u from the per-job unit bases (kernel parameters: no dependent memory load)
__device__ __forceinline__ int job_of(int u, int n_jobs, const int (&base)[kMaxJobs]) {
    int j = 0;
#pragma unroll
    for (int i = 1; i < kMaxJobs; ++i)
        if (i < n_jobs && u >= base[i]) j = i;
    return j;
}

template <int W>
struct MetaBlob {
    int32_t w[W];
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// per-thread 16-B async copy HBM -> SMEM (LDGSTS): no per-request copy-engine overhead, so it
// keeps up with HBM for sub-2-KB row slices where cp.async.bulk does not (scripts/microbench_stream.cu)
// (no L2::cache_hint operand: with it, ptxas 12.9 emitted for some expand instantiations an LDGSTS
// whose 64-bit descriptor sits in an odd uniform register -- "illegal instruction" at run time)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint64_t /*policy*/) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// L2 prefetch (no data returned to the SM).  Safe before griddepcontrol.wait even for lines a
// preceding kernel still writes: L2 is the point of coherence, the later real read sees them.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long gtime_raw() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// one thread waits on the preceding grid, the rest park at the barrier (a waiting
// griddepcontrol.wait polls and would steal issue slots from co-resident CTAs)
__device__ __forceinline__ void pdl_wait_cta() {
    if (threadIdx.x == 0) pdl_wait();
    __syncthreads();
}
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void stg128_na(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
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

// ------------------------------------------------------------------ element traits
template <typename T>
struct Elem;

template <>
struct Elem<__nv_bfloat16> {
    static constexpr int kVec = 8;
    static constexpr int kSize = 2;
    __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[kVec]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    // y (bf16) + d (fp32) -> one round-to-nearest-even to bf16
    __device__ __forceinline__ static uint4 add_round(const uint4& y, const float (&d)[kVec]) {
        float f[kVec];
        unpack(y, f);
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i] + d[2 * i], f[2 * i + 1] + d[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};

template <>
struct Elem<float> {
    static constexpr int kVec = 4;
    static constexpr int kSize = 4;
    __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[kVec]) {
        f[0] = __uint_as_float(v.x);
        f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z);
        f[3] = __uint_as_float(v.w);
    }
    __device__ __forceinline__ static uint4 add_round(const uint4& y, const float (&d)[kVec]) {
        return make_uint4(__float_as_uint(__uint_as_float(y.x) + d[0]), __float_as_uint(__uint_as_float(y.y) + d[1]),
                          __float_as_uint(__uint_as_float(y.z) + d[2]), __float_as_uint(__uint_as_float(y.w) + d[3]));
    }
};

// ------------------------------------------------------------------ metadata access
__device__ __forceinline__ int gc_field(const int32_t* M, int gc, int f) { return M[kHdrWords + gc * kGcFields + f]; }
// TP split (a.vred set, expand not yet run): the shrink CTA that completes a gc's partials sums them
// over the k-slices, in slice order, into the compact v [ntok][v_stride(r)] at GC_VRED -- the rank-r
// payload the TP ranks all-reduce (c5 decode: 15,360 B).  The CTA's own partial stores precede the
// counter increment (fence + barrier); the last arriver re-arms the counter for the next apply.
template <int NT>
__device__ __forceinline__ void tp_reduce_tail(const struct DecodeArgs& a, const int32_t* M, int gc, int* flag_smem);

// page of rank row j of a page reference (kernel_config.h page_ref_add)
__device__ __forceinline__ int page_at(const int32_t* M, int ref, int j) { return ref >= 0 ? M[ref + j] : (~ref) + j; }
// unit u's work record.  3-word mode: one round of independent uniform loads; 1-word mode (batches
// whose 3-word table would overflow the kernel parameters): the rest comes from the gc record.
struct UnitRec {
    int gc, local, pref, toff, r, ntok;
};
__device__ __forceinline__ UnitRec load_unit(const int32_t* M, int unit_tab, int unit_words, int u, bool shrink) {
    UnitRec d;
    const int32_t* rec = M + unit_tab + unit_words * u;
    const uint32_t uw = (uint32_t)rec[0];
    d.gc = (int)(uw >> 16);
    d.local = (int)(uw & 0xffffu);
    if (unit_words == 3) {
        const uint32_t rn = (uint32_t)rec[2];
        d.pref = rec[1];
        d.toff = unit_tok_off(rn);
        d.r = unit_rank(rn);
        d.ntok = unit_ntok(rn);
    } else {
        d.r = gc_field(M, d.gc, GC_RANK);
        d.ntok = gc_field(M, d.gc, GC_NTOK);
        d.toff = gc_field(M, d.gc, GC_TOK_OFF);
        d.pref = gc_field(M, d.gc, GC_PAGE_OFF);
        if (shrink) d.pref = page_ref_add(d.pref, (d.local % shrink_jblocks(d.r, 2)) * kShrinkRowsMma);
    }
    return d;
}

template <int NT>
__device__ __forceinline__ void tp_reduce_tail(const DecodeArgs& a, const int32_t* M, int gc, int* flag_smem) {
    const int tid = threadIdx.x;
    __threadfence();   // this thread's partial stores, gpu scope, before the counter
    __syncthreads();
    if (tid == 0) {
        const bool last_gc = gc + 1 >= a.n_gc;
        const int n_s = (last_gc ? a.n_shrink : gc_field(M, gc + 1, GC_SHRINK_BASE)) - gc_field(M, gc, GC_SHRINK_BASE);
        const int prev = atomicAdd(a.gc_cnt + gc, 1);
        *flag_smem = prev == n_s - 1;
        if (prev == n_s - 1) a.gc_cnt[gc] = 0;   // every shrink unit of the gc has arrived: re-arm
    }
    __syncthreads();
    if (!*flag_smem) return;
    __threadfence();   // acquire side: the other CTAs' partials
    const int r = gc_field(M, gc, GC_RANK), ntok = gc_field(M, gc, GC_NTOK), rs = v_stride(r);
    const int ksplit = a.jobs[gc_field(M, gc, GC_JOB)].ksplit;
    const float* src = a.vbuf + gc_field(M, gc, GC_VOFF);
    float* dst = a.vred + gc_field(M, gc, GC_VRED);
    for (int e = tid; e < ntok * rs; e += NT) {
        float v = 0.f;
        for (int k = 0; k < ksplit; ++k) v += ld_cg_f32(src + k * ntok * rs + e);
        dst[e] = v;
    }
}

// per-CTA unit description, decoded once by warp 0 and shared through smem
struct UnitSh {
    int job;
    int gc, r, ntok, ks, j0, nj, n0, nc, voff;
    float scale;
    int tok[kMaxTokChunk];
};

// ------------------------------------------------------------------ shrink kernel
// One CTA = one unit (group-chunk gc, k-slice ks, block of <= 8 rank rows): partial
// v[t][j0..j0+nj) over k in [k0, k0+nk) for the <= kTokChunk tokens of gc.
constexpr int kShrinkSmem = 256 + kShrinkRows * kSliceBytes + kTokChunk * kSliceBytes;   // 48.25 KB

template <typename T, int W>
__global__ void __launch_bounds__(kConsumerThreads)
    lora_shrink_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ MetaBlob<W> blob) {
    using E = Elem<T>;
    constexpr int V = E::kVec;
    constexpr int KS = kSliceBytes / E::kSize;
    extern __shared__ __align__(128) char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);          // [0] A rows, [1] x rows
    UnitSh* sh = reinterpret_cast<UnitSh*>(smem + 16);
    float* red = reinterpret_cast<float*>(smem + 128);            // kShrinkRows * kTokChunk floats
    char* abuf = smem + 256;
    char* xbuf = abuf + kShrinkRows * kSliceBytes;
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = blockIdx.x;
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 1] = gtime();
    if (W == 1) pdl_wait_cta();   // metadata uploaded by the preceding kernel

    int tok = 0;
    if (warp == 0) {
        // 1. decode the unit and issue the adapter-row loads (immutable pool pages) before
        //    waiting on the previous kernel in the stream
        const int job = job_of(u, a.n_jobs, a.job_shrink_base);
        const uint32_t uw = (uint32_t)M[a.unit_tab + a.unit_words * u];   // (gc, index in gc)
        const int gc = (int)(uw >> 16);
        const DecodeJob J = a.jobs[job];
        const int r = gc_field(M, gc, GC_RANK);
        const int ntok = gc_field(M, gc, GC_NTOK);
        const int local = (int)(uw & 0xffffu);
        const int poff = gc_field(M, gc, GC_PAGE_OFF);
        const int toff = gc_field(M, gc, GC_TOK_OFF);
        const int njb = shrink_jblocks(r, E::kSize);
        const int ks = local / njb;
        const int j0 = (local - ks * njb) * kShrinkRows;
        const int nj = min(kShrinkRows, r - j0);
        const int page = lane < nj ? page_at(M, poff, j0 + lane) : 0;
        tok = lane < ntok ? M[toff + lane] : 0;
        const int k0 = ks * KS;
        const uint32_t row_bytes = (uint32_t)min(KS, J.H_in - k0) * E::kSize;
        if (lane == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_arrive_expect_tx(&bars[0], (uint32_t)nj * row_bytes);
            sh->gc = gc; sh->job = job; sh->r = r; sh->ntok = ntok; sh->ks = ks; sh->j0 = j0; sh->nj = nj;
            sh->voff = gc_field(M, gc, GC_VOFF);
        }
        __syncwarp();
        if (lane < nj)
            bulk_g2s(abuf + lane * kSliceBytes, J.A + ((size_t)page * J.H_in + k0) * E::kSize, row_bytes,
                     &bars[0], policy_evict_first());
    }
    pdl_launch_dependents();
    __syncthreads();
    const DecodeJob J = a.jobs[sh->job];
    const int r = sh->r, ntok = sh->ntok, ks = sh->ks, j0 = sh->j0, nj = sh->nj;
    const int k0 = ks * KS;
    const int nk = min(KS, J.H_in - k0);
    // 2. x (and the v scratch we overwrite) may belong to the preceding kernel in the stream
    pdl_wait_cta();
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 2] = gtime();
    if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&bars[1], (uint32_t)(ntok * nk * E::kSize));
        __syncwarp();
        if (lane < ntok)
            bulk_g2s(xbuf + lane * kSliceBytes, J.x + ((size_t)tok * J.x_ld + k0) * E::kSize, (uint32_t)nk * E::kSize,
                     &bars[1], policy_evict_normal());
    }
    // 3. partial dot products: warp -> (row, k-part)
    const int P = kShrinkRows / nj;
    const int nit = (nk + 32 * V - 1) / (32 * V);
    const int ipp = (nit + P - 1) / P;
    mbar_wait(&bars[0], 0);
    mbar_wait(&bars[1], 0);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 3] = gtime();
    if (warp < nj * P) {
        const int row = warp % nj, part = warp / nj;
        float acc[kTokChunk];
#pragma unroll
        for (int t = 0; t < kTokChunk; ++t) acc[t] = 0.f;
        const char* arow = abuf + row * kSliceBytes;
        const int it1 = min(nit, (part + 1) * ipp);
#pragma unroll 4
        for (int it = part * ipp; it < it1; ++it) {
            const int e = (it * 32 + lane) * V;
            if (e < nk) {
                float av[V];
                E::unpack(lds128(arow + e * E::kSize), av);
#pragma unroll
                for (int t = 0; t < kTokChunk; ++t) {
                    if (t < ntok) {
                        float xv[V];
                        E::unpack(lds128(xbuf + t * kSliceBytes + e * E::kSize), xv);
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[t] = fmaf(xv[i], av[i], acc[t]);
                    }
                }
            }
        }
#pragma unroll
        for (int t = 0; t < kTokChunk; ++t) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < kTokChunk; ++t)
                if (t < ntok) red[(row * P + part) * kTokChunk + t] = acc[t];
        }
    }
    __syncthreads();
    const int padr = j0 + nj == r ? v_stride(r) - r : 0;   // zero tail of the row stride
    if (tid < (nj + padr) * ntok) {
        const int row = tid / ntok, t = tid - row * ntok;
        float v = 0.f;
        if (row < nj)
            for (int p = 0; p < P; ++p) v += red[(row * P + p) * kTokChunk + t];
        a.vbuf[sh->voff + (ks * ntok + t) * v_stride(r) + j0 + row] = v;
    }
    if (a.vred) tp_reduce_tail<kConsumerThreads>(a, M, sh->gc, &sh->ks);
    if (a.trace && tid == 0) {
        a.trace[(size_t)u * 8 + 0] = smid();
        a.trace[(size_t)u * 8 + 4] = sh->r;
        a.trace[(size_t)u * 8 + 5] = gtime();
    }
}

// ------------------------------------------------------------------ expand kernel
// One CTA = one unit (group-chunk gc, column slice [n0, n0+nc) of width ncols(r)):
// y[t][n0..n0+nc) += v[t][:] · B[:, n0..n0+nc) for the <= kTokChunk tokens of gc.
constexpr int kYBytes = kTokChunk * kConsumerThreads * 16;   // <= 4 tokens x 256 vectors x 16 B
constexpr int kExpandSmem = 256 + kTokChunk * LORA_MAX_RANK * 4 + kExpandBytes + kYBytes;

template <typename T, int W>
__global__ void __launch_bounds__(kConsumerThreads)
    lora_expand_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ MetaBlob<W> blob) {
    using E = Elem<T>;
    constexpr int V = E::kVec;
    extern __shared__ __align__(128) char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);          // [0] B rows, [1] y rows
    UnitSh* sh = reinterpret_cast<UnitSh*>(smem + 16);
    float* vsm = reinterpret_cast<float*>(smem + 256);            // [kTokChunk][r]
    char* bbuf = smem + 256 + kTokChunk * LORA_MAX_RANK * 4;      // [r][c] (reused as the reduction buffer)
    char* ybuf = bbuf + kExpandBytes;                             // [kTokChunk][c]
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ue = blockIdx.x;
    const int u = ue + a.n_shrink;
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 1] = gtime();
    if (W == 1) pdl_wait_cta();   // metadata uploaded by a preceding kernel

    int tok = 0;
    if (warp == 0) {
        // 1. decode the unit; B rows (immutable pool pages) before waiting on the shrink kernel
        const int job = job_of(ue, a.n_jobs, a.job_expand_base);
        const uint32_t uw = (uint32_t)M[a.unit_tab + a.unit_words * (a.n_shrink + ue)];
        const int gc = (int)(uw >> 16);
        const DecodeJob J = a.jobs[job];
        const int r = gc_field(M, gc, GC_RANK);
        const int ntok = gc_field(M, gc, GC_NTOK);
        const int local = (int)(uw & 0xffffu);
        const int poff = gc_field(M, gc, GC_PAGE_OFF);
        const int toff = gc_field(M, gc, GC_TOK_OFF);
        const int c = expand_ncols(r, E::kSize);
        const int n0 = local * c;
        const int nc = min(c, J.H_out - n0);
        int pages[LORA_MAX_RANK / 32];
#pragma unroll
        for (int q = 0; q < LORA_MAX_RANK / 32; ++q) pages[q] = (q * 32 + lane < r) ? page_at(M, poff, q * 32 + lane) : 0;
        tok = lane < ntok ? M[toff + lane] : 0;
        const uint32_t row_bytes = (uint32_t)nc * E::kSize;
        if (lane == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_arrive_expect_tx(&bars[0], (uint32_t)r * row_bytes);
            sh->gc = gc; sh->job = job; sh->r = r; sh->ntok = ntok; sh->n0 = n0; sh->nc = nc;
            sh->voff = gc_field(M, gc, GC_VOFF);
            sh->scale = __int_as_float(gc_field(M, gc, GC_SCALE));
        }
        if (lane < ntok) sh->tok[lane] = tok;
        __syncwarp();
        const uint64_t pol = policy_evict_first();
#pragma unroll
        for (int q = 0; q < LORA_MAX_RANK / 32; ++q) {
            const int j = q * 32 + lane;
            if (j < r)
                bulk_g2s(bbuf + (size_t)j * c * E::kSize, J.B + ((size_t)pages[q] * J.H_out + n0) * E::kSize,
                         row_bytes, &bars[0], pol);
        }
    }
    pdl_launch_dependents();
    __syncthreads();
    const DecodeJob J = a.jobs[sh->job];
    const int r = sh->r, ntok = sh->ntok, n0 = sh->n0, nc = sh->nc;
    const int c = expand_ncols(r, E::kSize);
    const size_t row_stride = (size_t)c * E::kSize;
    pdl_wait_cta();   // the shrink kernel's v (and y from whoever wrote it) are now visible
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 2] = gtime();
    if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&bars[1], (uint32_t)(ntok * nc * E::kSize));
        __syncwarp();
        if (lane < ntok)
            bulk_g2s(ybuf + lane * row_stride, J.y + ((size_t)tok * J.y_ld + n0) * E::kSize, (uint32_t)nc * E::kSize,
                     &bars[1], policy_evict_normal());
    }
    {
        // v: the k-slice partials summed in slice order, or the compact k-reduced v (TP split)
        const int voff = a.v_compact ? gc_field(M, sh->gc, GC_VRED) : sh->voff;
        const int ksplit = a.v_compact ? 1 : J.ksplit;
        const float* vsrc = a.v_compact ? a.vred : a.vbuf;
        const float scale = sh->scale;
        for (int i = tid; i < ntok * r; i += kConsumerThreads) {
            const int t = i / r, j = i - t * r;
            float v = 0.f;
            for (int k = 0; k < ksplit; ++k) v += ld_cg_f32(vsrc + voff + (k * ntok + t) * v_stride(r) + j);
            vsm[t * r + j] = v * scale;
        }
    }
    __syncthreads();
    mbar_wait(&bars[0], 0);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 3] = gtime();
    const int Cf = c / V;                   // vector columns of a full unit (power of two <= 256)
    const int P = kConsumerThreads / Cf;    // rank parts
    const int ci = tid % Cf, p = tid / Cf;
    const bool active = ci * V < nc;
    float acc[kTokChunk][V];
#pragma unroll
    for (int t = 0; t < kTokChunk; ++t)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[t][i] = 0.f;
    if (active) {
        const char* col = bbuf + ci * 16;
#pragma unroll 4
        for (int j = p; j < r; j += P) {
            float b[V];
            E::unpack(lds128(col + j * row_stride), b);
#pragma unroll
            for (int t = 0; t < kTokChunk; ++t) {
                if (t < ntok) {
                    const float vt = vsm[t * r + j];
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[t][i] = fmaf(vt, b[i], acc[t][i]);
                }
            }
        }
    }
    if (P == 1) {
        mbar_wait(&bars[1], 0);
        if (active) {
#pragma unroll
            for (int t = 0; t < kTokChunk; ++t) {
                if (t < ntok) {
                    const uint4 yo = lds128(ybuf + t * row_stride + ci * 16);
                    stg128_na(J.y + ((size_t)sh->tok[t] * J.y_ld + n0 + ci * V) * E::kSize, E::add_round(yo, acc[t]));
                }
            }
        }
    } else {
        // fixed-order reduction over the P rank parts, through the (now free) B buffer
        float* red = reinterpret_cast<float*>(bbuf);
        __syncthreads();
        if (active) {
#pragma unroll
            for (int t = 0; t < kTokChunk; ++t) {
                if (t < ntok) {
                    float* dst = red + ((size_t)(p * kTokChunk + t) * Cf + ci) * V;
#pragma unroll
                    for (int i = 0; i < V; i += 4)
                        *reinterpret_cast<float4*>(dst + i) =
                            make_float4(acc[t][i], acc[t][i + 1], acc[t][i + 2], acc[t][i + 3]);
                }
            }
        }
        __syncthreads();
        mbar_wait(&bars[1], 0);
        for (int it = tid; it < ntok * Cf; it += kConsumerThreads) {
            const int t = it / Cf, c2 = it - t * Cf;
            if (c2 * V >= nc) continue;
            float d[V];
#pragma unroll
            for (int i = 0; i < V; ++i) d[i] = 0.f;
            for (int q = 0; q < P; ++q) {
                const float* src = red + ((size_t)(q * kTokChunk + t) * Cf + c2) * V;
#pragma unroll
                for (int i = 0; i < V; ++i) d[i] += src[i];
            }
            const uint4 yo = lds128(ybuf + t * row_stride + c2 * 16);
            stg128_na(J.y + ((size_t)sh->tok[t] * J.y_ld + n0 + c2 * V) * E::kSize, E::add_round(yo, d));
        }
    }
    if (a.trace && tid == 0) {
        a.trace[(size_t)u * 8 + 0] = smid();
        a.trace[(size_t)u * 8 + 4] = sh->r;
        a.trace[(size_t)u * 8 + 5] = gtime();
    }
}

// ------------------------------------------------------------------ bf16 tensor-core (mma.sync) kernels
// The decode delta is HBM-bound; what limits a kernel that computes only after its data
// arrived is the chain after griddepcontrol.wait and how many adapter rows can be in flight
// before it (SMEM capacity).  The bf16 kernels therefore (a) stream every adapter row HBM -> SMEM
// before the wait (cp.async.bulk / LDGSTS) and read it once into mma.sync fragments (the shrink's
// A rows in the m16n8k16 layout up to a permutation of k that the x fragments repeat -- the dot
// product is order-free in k), (b) size their units so a q/k/v-sized grid is resident in one
// wave (6 shrink / 4 expand CTAs per SM), and (c) read the expand operand from shared memory
// exactly once (swap-AB: B^T tiles via ldmatrix.trans, each fragment feeding every token group).
// The MMA (fp32 accumulate) is a dot-product engine here: tiles are padded with zero rows (tokens
// to 8 N columns of (token, hi|lo) pairs, ranks to 16) in registers / smem only; HBM bytes are
// exactly the algorithmic ones.
constexpr int kPitchPad = 16;   // bytes added to each smem row: conflict-free ldmatrix

__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// D[16x8] += A[16x16] (row) * B[16x8] (col), bf16 inputs, fp32 accumulate
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint4 ldg_stream(const void* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ldg_cg128(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// ---- shrink (bf16): one CTA = (group-chunk gc, k-slice of kKSlice, 16 rank rows).  The rank
// rows go HBM -> SMEM with cp.async.bulk before griddepcontrol.wait (the copy engine, not the
// LSU: a co-resident CTA's critical-path loads/ldmatrix never queue behind this prefetch).
// Warp w owns k in [k0 + 128w, k0 + 128w + 128) as 4 blocks of 32; lane (g = lane/4,
// c = lane%4) reads rows g and g+8, elements [kb + 8c, kb + 8c + 8) of every block with one
// 128-bit shared load.  The MMA's logical k (2c, 2c+1 | 2c+8, 2c+9) maps to physical
// kb + 8c + (0,1 | 2,3) in MMA #1 and kb + 8c + (4,5 | 6,7) in MMA #2, for the A rows and the
// x rows alike (the dot product is order-free in k).
constexpr int kKPerWarp = kKSlice / kConsumerWarps;   // 128
constexpr int kKBlocks = kKPerWarp / 32;              // 4
constexpr int kAPitch = kKSlice * 2 + 64;             // bf16 row pitch: rows g, g+1 land 16 banks apart
// smem: [0,128) barrier + unit record | A rows [16][kAPitch] (reused for the warps' partial D tiles
// [8 warps][16 rows][8 tokens] fp32 once every warp has its A fragments in registers)
constexpr int kShrinkMmaSmem = 128 + kShrinkRowsMma * kAPitch;
static_assert(kConsumerWarps * kShrinkRowsMma * kTokChunkMma * 4 <= kShrinkRowsMma * kAPitch, "partials fit the A rows");
// Launch size of the bf16 shrink CTA (>= the ~33 KB it touches) sets how many shrink CTAs share an
// SM.  One pool per launch prefers 52 KB (4/SM: the grid spreads over more SMs; serial sweep
// 40 KB 89.9K, 52 KB 94.3K tok/s); grids of more than 4 CTAs per SM (q/k/v in one
// lora_apply_multi launch, 3x the units) take 34 KB (6/SM at <= 40 registers: more of the grid
// resident while the previous apply's expand CTAs still hold SMEM).
#ifndef LORA_X_PREFETCH
#define LORA_X_PREFETCH 1                         // shrink: L2 prefetch of the x rows before the PDL wait
#endif
#ifndef LORA_Y_PREFETCH
#define LORA_Y_PREFETCH 1                         // expand: L2 prefetch of the y rows before the PDL wait
#endif
#ifndef LORA_SHRINK_LAUNCH_KB
#define LORA_SHRINK_LAUNCH_KB 52                 // grids of <= 4 shrink CTAs per SM (one pool)
#endif
#ifndef LORA_SHRINK_LAUNCH_KB_BIG
#define LORA_SHRINK_LAUNCH_KB_BIG 34             // larger grids (q/k/v multi)
#endif
constexpr int kShrinkMmaLaunchSmem =
    kShrinkMmaSmem > LORA_SHRINK_LAUNCH_KB * 1024 ? kShrinkMmaSmem : LORA_SHRINK_LAUNCH_KB * 1024;
constexpr int kShrinkMmaLaunchSmemBig =
    kShrinkMmaSmem > LORA_SHRINK_LAUNCH_KB_BIG * 1024 ? kShrinkMmaSmem : LORA_SHRINK_LAUNCH_KB_BIG * 1024;

__device__ __forceinline__ void shrink_mma_body(const DecodeArgs& a, const int32_t* M, const int u, char* smem) {
    constexpr int ES = 2;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                    // [0] A rows
    UnitSh* sh = reinterpret_cast<UnitSh*>(smem + 16);
    char* abuf = smem + 128;                                               // [16 rows][kAPitch]
    float* part = reinterpret_cast<float*>(abuf);                          // [warp][16 rows][8 tokens] (after the A reads)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 0) {
        if (lane == 0) {   // barrier init first: its fence overlaps the metadata round trip
            mbar_init(&bars[0], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        const int job = job_of(u, a.n_jobs, a.job_shrink_base);
        // round 1: the unit record (independent uniform loads)
        const UnitRec ur = load_unit(M, a.unit_tab, a.unit_words, u, true);
        const int pg0 = ur.pref, toff = ur.toff;
        const int gc = ur.gc, local = ur.local;
        const int r = ur.r, ntok = ur.ntok;
        const DecodeJob J = a.jobs[job];
        const int njb = shrink_jblocks(r, ES);
        const int ks = local / njb;
        const int j0 = (local - ks * njb) * kShrinkRowsMma;
        const int nj = min(kShrinkRowsMma, r - j0);
        const int k0 = ks * kKSlice;
        const int nk = min(kKSlice, J.H_in - k0);
        // round 2: pages, tokens, v offset
        const int page = lane < nj ? page_at(M, pg0, lane) : 0;
        const int tokv = lane < ntok ? M[toff + lane] : -1;
        const int voff = gc_field(M, gc, GC_VOFF);
        if (a.trace) { asm volatile("" ::"r"(page), "r"(tokv)); if (lane == 0) a.trace[(size_t)u * 8 + 7] = gtime(); }
        if (lane < kTokChunkMma) sh->tok[lane] = tokv;
        if (LORA_X_PREFETCH && tokv >= 0) prefetch_l2(J.x + ((size_t)tokv * J.x_ld + k0) * ES, (uint32_t)(nk * ES));
        if (lane == 0) {
            mbar_arrive_expect_tx(&bars[0], (uint32_t)(nj * nk * ES));
            sh->gc = gc; sh->job = job; sh->r = r; sh->ntok = ntok; sh->ks = ks; sh->j0 = j0; sh->nj = nj;
            sh->voff = voff;
        }
        __syncwarp();
        if (lane < nj)
            bulk_g2s(abuf + lane * kAPitch, J.A + ((size_t)page * J.H_in + k0) * ES, (uint32_t)(nk * ES), &bars[0],
                     policy_evict_first());
    }
    pdl_launch_dependents();
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 6] = gtime();
    __syncthreads();
    const DecodeJob J = a.jobs[sh->job];
    const int g = lane >> 2, c = lane & 3;
    const int ks = sh->ks, ntok = sh->ntok, nj = sh->nj;
    const int k0 = ks * kKSlice;
    const int nk = min(kKSlice, J.H_in - k0);
    // x (and the v scratch we overwrite) may belong to the preceding kernel in the stream
    pdl_wait_cta();
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 2] = gtime();
    uint4 xr[kKBlocks];
    {
        const int tk = g < ntok ? sh->tok[g] : -1;
        const char* xrow = J.x + ((size_t)(tk < 0 ? 0 : tk) * J.x_ld + k0) * ES;
#pragma unroll
        for (int b = 0; b < kKBlocks; ++b) {
            const int k = warp * kKPerWarp + b * 32 + c * 8;
            xr[b] = (tk >= 0 && k < nk) ? ldg_cg128(xrow + k * ES) : make_uint4(0u, 0u, 0u, 0u);
        }
    }
    mbar_wait(&bars[0], 0);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 3] = gtime();
    // one accumulator chain over the warp's k-blocks (fixed order); A fragments loaded per k-block
    // (<= 40 registers: 6 CTAs per SM)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b < kKBlocks; ++b) {
        const int k = warp * kKPerWarp + b * 32 + c * 8;
        const bool kin = k < nk;
        const uint4 ra = (g < nj && kin) ? lds128(abuf + g * kAPitch + k * ES) : make_uint4(0u, 0u, 0u, 0u);
        const uint4 rb = (g + 8 < nj && kin) ? lds128(abuf + (g + 8) * kAPitch + k * ES) : make_uint4(0u, 0u, 0u, 0u);
        mma_bf16(acc, ra.x, rb.x, ra.y, rb.y, xr[b].x, xr[b].y);
        mma_bf16(acc, ra.z, rb.z, ra.w, rb.w, xr[b].z, xr[b].w);
    }
    __syncthreads();   // every warp's A reads done: the partial tiles reuse the A rows
    // D: (row g, tokens 2c, 2c+1) and (row g+8, tokens 2c, 2c+1)
    {
        float* pw = part + warp * kShrinkRowsMma * kTokChunkMma;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int row = g + ((q & 2) ? 8 : 0), t = 2 * c + (q & 1);
            pw[row * kTokChunkMma + t] = acc[q];
        }
    }
    __syncthreads();
    const int r = sh->r, j0 = sh->j0;
    const int padr = j0 + nj == r ? v_stride(r) - r : 0;   // zero tail of the row stride
    if (tid < (nj + padr) * ntok) {
        const int row = tid / ntok, t = tid - row * ntok;
        float v = 0.f;
        if (row < nj) {
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w) v += part[(w * kShrinkRowsMma + row) * kTokChunkMma + t];
        }
        a.vbuf[sh->voff + (ks * ntok + t) * v_stride(r) + j0 + row] = v;
    }
    if (a.vred) tp_reduce_tail<kConsumerThreads>(a, M, sh->gc, &sh->ks);
    if (a.trace && tid == 0) {
        a.trace[(size_t)u * 8 + 0] = smid();
        a.trace[(size_t)u * 8 + 4] = sh->r;
        a.trace[(size_t)u * 8 + 5] = gtime();
    }
}

template <int W>
__global__ void __launch_bounds__(kConsumerThreads, 6)
    lora_shrink_mma_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ MetaBlob<W> blob) {
    extern __shared__ __align__(128) char smem[];
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    if (a.trace && threadIdx.x == 0) a.trace[(size_t)blockIdx.x * 8 + 1] = gtime();
    if (W == 1) pdl_wait_cta();   // metadata uploaded by the preceding kernel
    shrink_mma_body(a, M, blockIdx.x, smem);
}

// ---- expand (bf16): one CTA = (group-chunk gc, column slice [n0, n0+nc)).  Swap-AB:
// D[col][n] = B^T[col][rank] · V[rank][n], M = 16 columns, N = 8, K = 16 ranks, where the 8 N
// columns are (token, part) pairs: v is split into bf16 hi + lo parts (so v keeps fp32-level
// accuracy) and each part is its own N column, D(col, t) = D[col][2t] + D[col][2t+1] -- one MMA per
// (tile, k-step) covers 4 tokens' hi and lo parts (a chunk of <= 4 tokens needs half the MMAs of a
// hi-MMA + lo-MMA scheme with tokens as N).  D is added into the y tile staged in smem (one rounding)
// and written back with 16-B stores.
// smem (per unit, kernel_config.h expand_mma_smem): [0,256) barriers + UnitSh | 64 zero bytes |
// V [token groups of 4][8 (token, part)][rp + 8] bf16 | B rows [r][c + 8] | y rows [ntok][c + 8] |
// D^T fp32 [ntok][c + 4] | pages [r]; c = the gc's unit width (GC_NCOLS).
#ifndef LORA_EXPAND_BULK_MIN
#define LORA_EXPAND_BULK_MIN 2048
#endif
constexpr int kBulkMinBytes = LORA_EXPAND_BULK_MIN;   // B row slices at least this long go through cp.async.bulk
#ifndef LORA_EXPAND_MINB
#define LORA_EXPAND_MINB 3                // expand CTAs per SM the register budget allows (experiments)
#endif
#ifndef LORA_EXPAND_BIG_MINB
#define LORA_EXPAND_BIG_MINB 4            // ... for grids of more than 3 expand CTAs per SM
#endif

// The expand MMAs of one unit: warp w owns 16-column tiles [TW w + 8 TW p, +TW) for passes p; per
// (tile, k-step) one ldmatrix.x4.trans of B^T feeds NG MMAs (token groups of 4: hi and lo parts as
// the N columns); D(col, t) = D[col][2t] + D[col][2t+1] goes to the fp32 staging tile dt.
template <int NG, int TW>
__device__ __forceinline__ void expand_mma_tiles(int ntiles, int ksteps, int r, int nc, int ntok, int warp, int aj, int an,
                                                 int g, int cc, uint32_t zaddr, uint32_t v_base, int vpitch,
                                                 uint32_t b_base, int bpitch, float* dt, int dpitch) {
    constexpr int ES = 2;
#pragma unroll 1
    for (int tile0 = warp * TW; tile0 < ntiles; tile0 += kConsumerWarps * TW) {
        float d[NG][TW][4];
#pragma unroll
        for (int q = 0; q < NG; ++q)
#pragma unroll
            for (int i = 0; i < TW; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) d[q][i][e] = 0.f;
        for (int s = 0; s < ksteps; ++s) {
            const int j = s * 16 + aj;
            uint32_t v[NG][2], af[TW][4];
#pragma unroll
            for (int q = 0; q < NG; ++q) ldsm_x2(v[q][0], v[q][1], v_base + q * 8 * vpitch + s * 32);
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const int col = (tile0 + i) * 16 + an;
                ldsm_x4_trans(af[i][0], af[i][1], af[i][2], af[i][3],
                              (j < r && tile0 + i < ntiles) ? b_base + j * bpitch + col * ES : zaddr);
            }
#pragma unroll
            for (int q = 0; q < NG; ++q)
#pragma unroll
                for (int i = 0; i < TW; ++i) mma_bf16(d[q][i], af[i][0], af[i][1], af[i][2], af[i][3], v[q][0], v[q][1]);
        }
        // D^T (hi + lo) -> fp32 [token][col] staging (its own region: no barrier against B readers)
#pragma unroll
        for (int q = 0; q < NG; ++q) {
            const int t = q * 4 + cc;
            if (t < ntok) {
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    const int n = (tile0 + i) * 16 + g;
                    if (n < nc) dt[t * dpitch + n] = d[q][i][0] + d[q][i][1];
                    if (n + 8 < nc) dt[t * dpitch + n + 8] = d[q][i][2] + d[q][i][3];
                }
            }
        }
    }
}

__device__ __forceinline__ void expand_mma_body(const DecodeArgs& a, const int32_t* M, const int ue, char* smem) {
    constexpr int ES = 2;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);          // [0] B rows, [1] y rows
    UnitSh* sh = reinterpret_cast<UnitSh*>(smem + 16);
    char* zero = smem + 256;                                      // 64 zero bytes
    char* vt_s = smem + 320;                                      // V [ngrp][8][vpitch] bf16
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = ue + a.n_shrink;

    int tok = 0;
    if (warp == 0) {
        // 1. decode the unit; B rows (immutable pool pages) before waiting on the shrink kernel
        if (lane == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        const int job = job_of(ue, a.n_jobs, a.job_expand_base);
        const UnitRec ur = load_unit(M, a.unit_tab, a.unit_words, a.n_shrink + ue, false);
        const int poff = ur.pref, toff = ur.toff;
        const int gc = ur.gc, local = ur.local;
        const int r = ur.r, ntok = ur.ntok;
        const DecodeJob J = a.jobs[job];
        const int c = gc_field(M, gc, GC_NCOLS);
        const int n0 = local * c;
        const int nc = min(c, J.H_out - n0);
        const int bpitch = c * ES + kPitchPad;
        char* bbuf = smem + expand_mma_boff(r, ntok);
        int* spages = reinterpret_cast<int*>(smem + expand_mma_smem(r, c, ntok) - r * 4);
        int pages[LORA_MAX_RANK / 32];
#pragma unroll
        for (int q = 0; q < LORA_MAX_RANK / 32; ++q) pages[q] = (q * 32 + lane < r) ? page_at(M, poff, q * 32 + lane) : 0;
        tok = lane < ntok ? M[toff + lane] : 0;
        const uint32_t row_bytes = (uint32_t)nc * ES;
        const bool bulk = row_bytes >= kBulkMinBytes;
        if (lane == 0) {
            if (bulk) mbar_arrive_expect_tx(&bars[0], (uint32_t)r * row_bytes);
            sh->gc = gc; sh->job = job; sh->r = r; sh->ntok = ntok; sh->n0 = n0; sh->nc = nc; sh->j0 = c;
            sh->voff = gc_field(M, gc, GC_VOFF);
            sh->scale = __int_as_float(gc_field(M, gc, GC_SCALE));
        }
        if (lane < ntok) {
            sh->tok[lane] = tok;
            if (LORA_Y_PREFETCH) prefetch_l2(J.y + ((size_t)tok * J.y_ld + n0) * ES, row_bytes);
        }
        if (lane < 16) reinterpret_cast<uint32_t*>(zero)[lane] = 0u;
        __syncwarp();
        const uint64_t pol = policy_evict_first();
        if (bulk) {
#pragma unroll
            for (int q = 0; q < LORA_MAX_RANK / 32; ++q) {
                const int j = q * 32 + lane;
                if (j < r)
                    bulk_g2s(bbuf + (size_t)j * bpitch, J.B + ((size_t)pages[q] * J.H_out + n0) * ES, row_bytes,
                             &bars[0], pol);
            }
        } else {
#pragma unroll
            for (int q = 0; q < LORA_MAX_RANK / 32; ++q)
                if (q * 32 + lane < r) spages[q * 32 + lane] = pages[q];
        }
    }
    __syncthreads();
    const DecodeJob J = a.jobs[sh->job];
    const int r = sh->r, ntok = sh->ntok, n0 = sh->n0, nc = sh->nc;
    const int c = sh->j0;                   // the gc's unit width
    const int bpitch = c * ES + kPitchPad;
    const int ypitch = c * ES + kPitchPad;
    const int rp = (r + 15) & ~15;
    const int vpitch = (rp + 8) * 2;
    char* bbuf = smem + expand_mma_boff(r, ntok);
    char* ybuf = bbuf + r * bpitch;
    float* dt = reinterpret_cast<float*>(ybuf + ntok * ypitch);   // [ntok][nc + 4]
    const int* spages = reinterpret_cast<const int*>(smem + expand_mma_smem(r, c, ntok) - r * 4);
    const bool bulk = nc * ES >= kBulkMinBytes;
    if (!bulk) {
        // sub-2-KB row slices: every thread streams 16-B pieces (a warp covers 512 contiguous bytes)
        const uint64_t pol = policy_evict_first();
        const int vpr = nc / 8;
        for (int i = tid; i < r * vpr; i += kConsumerThreads) {
            const int j = i / vpr, q = i - j * vpr;
            cp_async16(bbuf + (size_t)j * bpitch + q * 16, J.B + ((size_t)spages[j] * J.H_out + n0 + q * 8) * ES, pol);
        }
        cp_async_commit();
    }
    pdl_launch_dependents();
    pdl_wait_cta();   // v from the shrink kernel, y from whoever wrote it
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 2] = gtime();
    if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&bars[1], (uint32_t)(ntok * nc * ES));
        __syncwarp();
        if (lane < ntok)
            bulk_g2s(ybuf + lane * ypitch, J.y + ((size_t)tok * J.y_ld + n0) * ES, (uint32_t)nc * ES, &bars[1],
                     policy_evict_normal());
    }
    const int ngrp = (ntok + 3) >> 2;       // token groups of 4: one MMA each per (tile, k-step)
    // v (fp32, summed over k-slices, scaled) -> bf16 (hi, lo) rows: token t = 4 grp + tl at rows
    // [grp][2 tl] (hi) and [grp][2 tl + 1] (lo)
    {
        // v: the k-slice partials summed in slice order, or the compact k-reduced v (TP split)
        const int voff = a.v_compact ? gc_field(M, sh->gc, GC_VRED) : sh->voff;
        const int ksplit = a.v_compact ? 1 : J.ksplit;
        const float* vsrc = a.v_compact ? a.vred : a.vbuf;
        const float scale = sh->scale;
        for (int i = tid; i < 4 * ngrp * rp; i += kConsumerThreads) {
            const int t = i / rp, j = i - t * rp;
            float v = 0.f;
            if (t < ntok && j < r) {
                // k-slice partials: batches of 8 independent loads, summed in slice order
                const float* src = vsrc + voff + t * v_stride(r) + j;
                const int stride = ntok * v_stride(r);
                for (int k0 = 0; k0 < ksplit; k0 += 8) {
                    float p[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) p[q] = k0 + q < ksplit ? ld_cg_f32(src + (k0 + q) * stride) : 0.f;
#pragma unroll
                    for (int q = 0; q < 8; ++q) v += p[q];
                }
                v *= scale;
            }
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
            char* row = vt_s + ((t >> 2) * 8 + 2 * (t & 3)) * vpitch + j * 2;
            *reinterpret_cast<__nv_bfloat16*>(row) = h;
            *reinterpret_cast<__nv_bfloat16*>(row + vpitch) = l;
        }
    }
    if (!bulk) cp_async_wait_all();
    __syncthreads();
    if (bulk) mbar_wait(&bars[0], 0);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 3] = gtime();
    const int ntiles = (nc + 15) / 16;
    const int ksteps = rp / 16;
    // A operand (B^T) via ldmatrix.x4.trans: matrix m = lane/8, row i = lane%8 -> rank j, column n
    const int am = lane >> 3, ai = lane & 7;
    const int aj = ai + ((am & 2) ? 8 : 0), an = (am & 1) * 8;
    // B operand (V): lanes 0-7 rows (token, part) at rank j, lanes 8-15 at j+8
    const int vn = lane & 7, vh = (lane >> 3) & 1;
    const uint32_t zaddr = smem_u32(zero);
    const uint32_t v_base = smem_u32(vt_s) + vn * vpitch + vh * 16;
    const uint32_t b_base = smem_u32(bbuf);
    const int g = lane >> 2, cc = lane & 3;   // D: column g (+8), N columns 2cc (hi), 2cc+1 (lo) = token cc
    const int dpitch = nc + 4;
    // chunks of <= 4 tokens: one token group, 4 column tiles per warp pass; 5..8 tokens: both groups
    // share every B fragment (2 MMAs per ldmatrix), 2 tiles per pass (same accumulator registers)
    if (ngrp == 1)
        expand_mma_tiles<1, 4>(ntiles, ksteps, r, nc, ntok, warp, aj, an, g, cc, zaddr, v_base, vpitch, b_base, bpitch,
                               dt, dpitch);
    else
        expand_mma_tiles<2, 2>(ntiles, ksteps, r, nc, ntok, warp, aj, an, g, cc, zaddr, v_base, vpitch, b_base, bpitch,
                               dt, dpitch);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 7] = gtime();
    mbar_wait(&bars[1], 0);
    if (a.trace && tid == 0) a.trace[(size_t)u * 8 + 6] = gtime();
    __syncthreads();
    {
        const int vpr = nc / 8;   // 16-B vectors per token row
        for (int i = tid; i < ntok * vpr; i += kConsumerThreads) {
            const int t = i / vpr, q = i - t * vpr;
            const float4 d0 = *reinterpret_cast<const float4*>(dt + t * dpitch + q * 8);
            const float4 d1 = *reinterpret_cast<const float4*>(dt + t * dpitch + q * 8 + 4);
            const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
            const uint4 yo = lds128(ybuf + t * ypitch + q * 16);
            stg128_na(J.y + ((size_t)sh->tok[t] * J.y_ld + n0 + q * 8) * ES, Elem<__nv_bfloat16>::add_round(yo, d));
        }
    }
    if (a.trace && tid == 0) {
        a.trace[(size_t)u * 8 + 0] = smid();
        a.trace[(size_t)u * 8 + 4] = sh->r;
        a.trace[(size_t)u * 8 + 5] = gtime();
    }
}

// MINB: CTAs per SM the register budget allows (3: <= 85 registers; 4: <= 64, no spills) -- the
// launcher takes 4 only for grids of more than 3 expand CTAs per SM (q/k/v multi launches)
template <int W, int MINB = LORA_EXPAND_MINB>
__global__ void __launch_bounds__(kConsumerThreads, MINB)
    lora_expand_mma_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ MetaBlob<W> blob) {
    extern __shared__ __align__(128) char smem[];
    const int32_t* M = (W > 1) ? blob.w : a.meta_global;
    if (a.trace && threadIdx.x == 0) a.trace[(size_t)(blockIdx.x + a.n_shrink) * 8 + 1] = gtime();
    if (W == 1) pdl_wait_cta();
    expand_mma_body(a, M, blockIdx.x, smem);
}

// copies a metadata blob too large for one kernel's parameters into device memory,
// kUploadWords per launch (parameters are captured by value in CUDA graphs)
constexpr int kUploadWords = 7936;
__global__ void lora_meta_upload_kernel(int32_t* dst, const __grid_constant__ MetaBlob<kUploadWords> b, int n) {
    pdl_wait_cta();
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = b.w[i];
}

// ------------------------------------------------------------------ host launcher
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, int grid, int block, int smem, cudaStream_t st, Args... args) {
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

// bf16 pools take the tensor-core (mma.sync) kernels, fp32 pools the SIMT FFMA kernels
// (TF32 would miss the 1e-5 fp32 bound).
template <typename T, int W>
struct DecodeKernels {
    static constexpr auto shrink = lora_shrink_kernel<T, W>;
    static constexpr auto expand = lora_expand_kernel<T, W>;
    static constexpr auto expand_big = lora_expand_kernel<T, W>;    // unused (== expand)
    static constexpr int shrink_smem = kShrinkSmem;
    static constexpr int shrink_smem_big = kShrinkSmem;
    static int expand_launch_smem(const DecodeArgs&) { return kExpandSmem; }
};
template <int W>
struct DecodeKernels<__nv_bfloat16, W> {
    static constexpr auto shrink = lora_shrink_mma_kernel<W>;
    static constexpr auto expand = lora_expand_mma_kernel<W>;
    static constexpr auto expand_big = lora_expand_mma_kernel<W, LORA_EXPAND_BIG_MINB>;
    static constexpr int shrink_smem = kShrinkMmaLaunchSmem;
    static constexpr int shrink_smem_big = kShrinkMmaLaunchSmemBig;
    static int expand_launch_smem(const DecodeArgs& a) { return a.e_smem; }
};

// cudaFuncSetAttribute is per device: one bit per (instantiation, device)
static bool configure_once(std::atomic<uint64_t>& mask, cudaError_t (*fn)()) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return fn() == cudaSuccess;
    const uint64_t bit = 1ull << dev;
    if (mask.load(std::memory_order_acquire) & bit) return true;
    if (fn() != cudaSuccess) return false;
    mask.fetch_or(bit, std::memory_order_acq_rel);
    return true;
}

template <typename T, int W>
static cudaError_t launch_pair(const DecodeArgs& a, const Plan& pl, cudaStream_t st, int* launches, int phases,
                               int num_sms) {
    using K = DecodeKernels<T, W>;
    static std::atomic<uint64_t> configured{0};
    if (!configure_once(configured, [] {
            // the opt-in maximum (the launch passes the real size; it decides occupancy)
            constexpr int kMaxOptin = 227 * 1024;
            cudaError_t e = cudaFuncSetAttribute(K::shrink, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxOptin);
            if (e == cudaSuccess) e = cudaFuncSetAttribute(K::expand, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxOptin);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(K::expand_big, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxOptin);
            return e;
        }))
        return cudaErrorInvalidValue;
    MetaBlob<W> blob;
    if (W > 1) {
        const int n = (int)pl.blob.size();
        for (int i = 0; i < n; ++i) blob.w[i] = pl.blob[i];
    }
    cudaError_t e = cudaSuccess;
    if (phases & 1) {
        // bf16: a grid of more than 4 shrink CTAs per SM (e.g. q/k/v in one multi launch) fits better
        // at 5 per SM (DESIGN.md §6 N1 occupancy)
        const int ss = pl.n_shrink > 4 * num_sms ? K::shrink_smem_big : K::shrink_smem;
        e = launch_pdl(K::shrink, pl.n_shrink, kConsumerThreads, ss, st, a, blob);
        if (e != cudaSuccess) return e;
        *launches += 1;
    }
    if (phases & 2) {
        const bool big = pl.n_expand > 3 * num_sms;
        e = launch_pdl(big ? K::expand_big : K::expand, pl.n_expand, kConsumerThreads, K::expand_launch_smem(a), st, a,
                       blob);
        *launches += 1;
    }
    return e;
}

template <typename T>
static cudaError_t launch_typed(const Plan& pl, const DecodeLaunch& L, cudaStream_t st, int* launches) {
    DecodeArgs a;
    memset(&a, 0, sizeof(a));
    for (int j = 0; j < L.n_jobs && j < kMaxJobs; ++j) {
        const void* x = j == 0 ? L.x : L.more[j - 1].x;
        void* y = j == 0 ? L.y : L.more[j - 1].y;
        const void* A = j == 0 ? L.poolA : L.more[j - 1].poolA;
        const void* B = j == 0 ? L.poolB : L.more[j - 1].poolB;
        const int hin = j == 0 ? L.H_in : L.more[j - 1].H_in, hout = j == 0 ? L.H_out : L.more[j - 1].H_out;
        const int xld = j == 0 && L.x_ld > 0 ? (int)L.x_ld : hin, yld = j == 0 && L.y_ld > 0 ? (int)L.y_ld : hout;
        a.jobs[j] = DecodeJob{static_cast<const char*>(x), static_cast<char*>(y), static_cast<const char*>(A),
                              static_cast<const char*>(B), hin, hout, ksplit_of(hin, (int)sizeof(T)), xld, yld};
    }
    a.vbuf = L.vbuf;
    a.v_compact = (L.phases == 2 && L.vred) ? 1 : 0;
    a.vred = (L.phases == 1 && !L.gc_cnt) ? nullptr : L.vred;   // the shrink's reduce tail needs the counters
    a.gc_cnt = L.gc_cnt;
    a.meta_global = L.meta_dev;
    a.trace = L.trace;
    a.n_shrink = pl.n_shrink;
    a.n_expand = pl.n_expand;
    a.n_gc = pl.n_gc;
    a.unit_tab = pl.unit_tab;
    a.unit_words = pl.unit_words;
    a.n_jobs = pl.n_jobs;
    for (int j = 0; j < kMaxJobs; ++j) {
        a.job_shrink_base[j] = pl.job_shrink_base[j];
        a.job_expand_base[j] = pl.job_expand_base[j];
    }
    if (sizeof(T) == 2) {
        // bf16 expand: every CTA lays out its own unit (expand_mma_smem); the launch reserves the largest
        int e_smem = 0;
        for (int gc = 0; gc < pl.n_gc; ++gc) {
            const int32_t* e = pl.blob.data() + kHdrWords + kGcFields * gc;
            const int need = expand_mma_smem(e[GC_RANK], e[GC_NCOLS], e[GC_NTOK]);
            e_smem = need > e_smem ? need : e_smem;
        }
        a.e_smem = e_smem;
    }
    const int n = (int)pl.blob.size();
    if (n <= 1024) return launch_pair<T, 1024>(a, pl, st, launches, L.phases, L.num_sms);
    if (n <= 2048) return launch_pair<T, 2048>(a, pl, st, launches, L.phases, L.num_sms);
    if (n <= 4096) return launch_pair<T, 4096>(a, pl, st, launches, L.phases, L.num_sms);
    if (n <= kUploadWords) return launch_pair<T, kUploadWords>(a, pl, st, launches, L.phases, L.num_sms);
    for (int off = 0; off < n && (L.phases & 1); off += kUploadWords) {   // expand-only reuses the shrink's upload
        const int m = n - off < kUploadWords ? n - off : kUploadWords;
        MetaBlob<kUploadWords> b;
        for (int i = 0; i < m; ++i) b.w[i] = pl.blob[off + i];
        cudaError_t e = launch_pdl(lora_meta_upload_kernel, 1, 256, 0, st, L.meta_dev + off, b, m);
        *launches += 1;
        if (e != cudaSuccess) return e;
    }
    return launch_pair<T, 1>(a, pl, st, launches, L.phases, L.num_sms);
}

int launch_decode(const Plan& pl, const DecodeLaunch& L, cudaStream_t st, int* launches) {
    if (L.esz == 2) return (int)launch_typed<__nv_bfloat16>(pl, L, st, launches);
    return (int)launch_typed<float>(pl, L, st, launches);
}

}  // namespace lora
