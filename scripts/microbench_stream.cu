// Streaming-read microbenchmark on sm_100a: HBM -> SMEM via cp.async.bulk in pieces of P
// bytes (one producer thread per CTA, S-stage ring of 32 KB) vs plain LDG.128 loops.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ms scripts/microbench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kStages = 4;
constexpr int kStage = 32768;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const char* src, size_t bytes_per_cta, int piece, unsigned long long* sink) {
    extern __shared__ __align__(128) char sm[];
    uint64_t* full = (uint64_t*)(sm + kStages * kStage);
    const char* base = src + (size_t)blockIdx.x * bytes_per_cta;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long acc = 0;
    const int nst = (int)(bytes_per_cta / kStage);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int per = kStage / piece;
        for (int it = 0; it < nst + kStages; ++it) {
            const int s = it % kStages;
            if (it >= kStages) {   // consume stage s from iteration it - kStages
                const uint32_t par = ((it - kStages) / kStages) & 1;
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(&full[s])), "r"(par));
                acc += *(volatile uint32_t*)(sm + s * kStage + lane * 4);
            }
            if (it < nst) {
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kStage));
                __syncwarp();
                for (int q = lane; q < per; q += 32)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     sa(sm + s * kStage + q * piece)),
                                 "l"(base + (size_t)it * kStage + (size_t)q * piece), "r"(piece), "r"(sa(&full[s]))
                                 : "memory");
            }
        }
    }
    if (acc == 123456789ull) sink[0] = acc;
}

__global__ void k_ldg(const int4* src, size_t vec_per_cta, unsigned long long* sink) {
    const int4* base = src + (size_t)blockIdx.x * vec_per_cta;
    int acc = 0;
    for (size_t i = threadIdx.x; i < vec_per_cta; i += blockDim.x * 8) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i + u * blockDim.x < vec_per_cta ? __ldg(base + i + u * blockDim.x) : int4{0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 123456789) sink[0] = acc;
}

int main() {
    const size_t total = (size_t)1 << 30;   // 1 GiB read per launch (>> L2)
    char* src;
    unsigned long long* sink;
    cudaMalloc(&src, total);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 1, total);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage + 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ctas_per_sm : {1, 2, 4}) {
        for (int piece : {512, 2048, 8192, 32768}) {
            const int grid = 148 * ctas_per_sm;
            const size_t per = (total / grid) / kStage * kStage;
            k_bulk<<<grid, 64, kStages * kStage + 64>>>(src, per, piece, sink);
            cudaEventRecord(e0);
            for (int r = 0; r < 3; ++r) k_bulk<<<grid, 64, kStages * kStage + 64>>>(src, per, piece, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("bulk ctas/SM=%d piece=%6d: %7.1f GB/s (%s)\n", ctas_per_sm, piece, 3.0 * per * grid / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int grid : {148, 296, 592, 1184}) {
        const size_t vec = total / 16 / grid;
        k_ldg<<<grid, 256>>>((const int4*)src, vec, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) k_ldg<<<grid, 256>>>((const int4*)src, vec, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg grid=%5d x256: %7.1f GB/s\n", grid, 3.0 * vec * 16 * grid / (ms * 1e-3) / 1e9);
    }
    return 0;
}
