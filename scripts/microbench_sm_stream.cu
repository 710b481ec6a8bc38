// Per-SM streaming ceiling on sm_100a: how many GB/s one CTA per SM moves HBM -> SM with
//   tma   : cp.async.bulk (1-D, 16 KB pieces) into an S-stage ring, one producer lane
//   ldg   : LDG.128 by all threads, U independent loads in flight per thread
//   mix   : half the CTA's bytes by the TMA ring, half by LDG warps, concurrently
//   rmw   : TMA read of y pieces + STG write back of the same bytes (the prefill y pattern)
//   rmwl  : LDG read + STG write (same bytes)
// Grid = G CTAs (1 per SM), each streaming its own BPC bytes; L2 is flushed before each run.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mss scripts/microbench_sm_stream.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPiece = 16384;
constexpr int kMaxStages = 12;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bwait(uint32_t bar, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar), "r"(par)
                 : "memory");
}

// mode 0 tma, 1 ldg, 2 mix, 3 rmw (tma read + stg write), 4 rmwl (ldg read + stg write)
__global__ void __launch_bounds__(256, 1) k_stream(char* buf, size_t bpc, int mode, int stages, unsigned long long* sink) {
    extern __shared__ __align__(1024) char sm[];
    uint64_t* full = (uint64_t*)(sm + kMaxStages * kPiece);
    char* base = buf + (size_t)blockIdx.x * bpc;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kMaxStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long acc = 0;
    size_t tma_bytes = (mode == 0 || mode == 3) ? bpc : (mode == 2 ? bpc / 2 : 0);
    size_t ldg_lo = (mode == 2) ? bpc / 2 : 0;
    size_t ldg_bytes = (mode == 1 || mode == 4) ? bpc : (mode == 2 ? bpc / 2 : 0);
    if (tma_bytes && warp == 0) {
        // producer lane + consumer (warp 0 consumes: touches one word, or writes the piece back)
        const int n = (int)(tma_bytes / kPiece);
        for (int it = 0; it < n + stages; ++it) {
            const int s = it % stages;
            if (it >= stages) {
                const int c = it - stages;
                bwait(sa(&full[s]), (uint32_t)((c / stages) & 1));
                if (mode == 3) {   // write the piece back (y RMW pattern): 16 KB by 32 lanes
                    const uint4* src = (const uint4*)(sm + s * kPiece);
                    uint4* dst = (uint4*)(base + (size_t)c * kPiece);
#pragma unroll 8
                    for (int i = lane; i < kPiece / 16; i += 32) dst[i] = src[i];
                } else {
                    acc += *(volatile uint32_t*)(sm + s * kPiece + lane * 4);
                }
                __syncwarp();
            }
            if (it < n && lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kPiece));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(sm + s * kPiece)),
                    "l"(base + (size_t)it * kPiece), "r"(kPiece), "r"(sa(&full[s]))
                    : "memory");
            }
            __syncwarp();
        }
    }
    if (ldg_bytes) {
        // LDG warps: all 8 warps in ldg/rmwl, warps 1..7 in mix
        const int w0 = (mode == 2) ? 1 : 0;
        if (warp >= w0) {
            const int nthr = (8 - w0) * 32, t = tid - w0 * 32;
            const uint4* p = (const uint4*)(base + ldg_lo);
            uint4* q = (uint4*)(base + ldg_lo);
            const size_t nv = ldg_bytes / 16;
            constexpr int U = 8;
            size_t i = t;
            for (; i + (U - 1) * nthr < nv; i += U * nthr) {
                uint4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * nthr);
                if (mode == 4) {
#pragma unroll
                    for (int u = 0; u < U; ++u) q[i + u * nthr] = v[u];
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
                }
            }
        }
    }
    if (acc == 0x1234567) sink[0] = acc;
}

// read-only flush: evicts the previous run's lines without leaving dirty lines in L2 (a writing
// flush makes the next "read-only" run pay ~L2-size of write-backs)
__global__ void k_flush(const char* p, size_t n, unsigned long long* sink) {
    unsigned acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 16; i += (size_t)gridDim.x * blockDim.x)
        acc ^= __ldcg((const uint4*)p + i).x;
    if (acc == 0x1234567u) sink[0] = acc;
}

int main() {
    const size_t flush_n = 512ull << 20;
    char *buf, *fl;
    unsigned long long* sink;
    const size_t bpc = 2ull << 20;
    cudaMalloc(&buf, bpc * 296);
    cudaMalloc(&fl, flush_n);
    cudaMemset(fl, 0, flush_n);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, bpc * 296);
    const int smem = kMaxStages * kPiece + 1024;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[5] = {"tma ", "ldg ", "mix ", "rmw ", "rmwl"};
    for (int grid : {128, 148}) {
        for (int mode = 0; mode < 5; ++mode) {
            for (int stages : {6, 12}) {
                if ((mode == 1 || mode == 4) && stages != 12) continue;
                float best = 1e9f;
                for (int rep = 0; rep < 5; ++rep) {
                    k_flush<<<592, 512>>>(fl, flush_n, sink);
                    if (mode >= 3) k_flush<<<592, 512>>>(fl, flush_n, sink);
                    cudaEventRecord(a);
                    k_stream<<<grid, 256, smem>>>(buf, bpc, mode, stages, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                const double moved = (double)bpc * grid * ((mode >= 3) ? 2.0 : 1.0);
                printf("grid %3d %s stages %2d: %7.2f us  %7.1f GB/s chip  %6.1f GB/s per SM (bytes %s)\n", grid,
                       names[mode], stages, best * 1e3, moved / (best * 1e-3) / 1e9, moved / (best * 1e-3) / 1e9 / grid,
                       mode >= 3 ? "read+write" : "read");
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
