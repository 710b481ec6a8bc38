// Microbenchmark of per-SM instruction costs on sm_100a: legacy HMMA (mma.sync m16n8k16
// bf16), LDSM (ldmatrix), FFMA, and globaltimer/clock64 granularity.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_sm.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void k_hmma(int iters, long long* out, float* sink) {
    float d[CHAINS][4] = {};
    uint32_t a = threadIdx.x * 0x3f803f80u, b = 0x3f803f80u;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) mma(d[c], a, a, a, a, b, b);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += d[c][0];
    if (s == 12345.f) sink[0] = s;
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

__global__ void k_ldsm(int iters, long long* out, float* sink) {
    __shared__ __align__(128) char buf[16384];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) ((uint32_t*)buf)[i] = i;
    __syncthreads();
    uint32_t addr = (uint32_t)__cvta_generic_to_shared(buf) + (threadIdx.x & 31) * 16 * 33 % 16384;
    addr &= ~15u;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r0, r1, r2, r3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(addr));
        acc ^= r0 ^ r3;
    }
    long long t1 = clock64();
    if (acc == 0x12345) sink[0] = acc;
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

__global__ void k_ffma(int iters, long long* out, float* sink) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], 1.0001f, 0.5f);
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.f) sink[0] = s;
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

__global__ void k_timer(unsigned long long* out) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(prev));
    int n = 0;
    unsigned long long mind = ~0ull;
    for (int i = 0; i < 200000 && n < 64; ++i) {
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        if (t != prev) {
            if (t - prev < mind) mind = t - prev;
            prev = t;
            ++n;
        }
    }
    out[0] = mind;
}

template <typename K>
void run(const char* name, K kern, int warps, int iters, int per_iter_instr, int blocks = 148) {
    long long* d_out;
    float* sink;
    cudaMalloc(&d_out, sizeof(long long) * blocks * 32);
    cudaMalloc(&sink, 4);
    cudaMemset(d_out, 0, sizeof(long long) * blocks * 32);
    kern<<<blocks, warps * 32>>>(iters, d_out, sink);
    kern<<<blocks, warps * 32>>>(iters, d_out, sink);
    cudaDeviceSynchronize();
    long long h[148 * 32];
    cudaMemcpy(h, d_out, sizeof(long long) * blocks * 32, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int w = 0; w < warps; ++w) avg += h[w];
    avg /= warps;
    printf("%-28s warps/SM=%2d  cycles/iter/warp=%7.2f  => %.2f cycles per instr per warp (%s)\n", name, warps,
           avg / iters, avg / iters / per_iter_instr, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d_out);
    cudaFree(sink);
}

int main() {
    for (int w : {1, 4, 8, 16}) {
        run("hmma 1 chain", k_hmma<1>, w, 2000, 1);
        run("hmma 8 chains", k_hmma<8>, w, 500, 8);
    }
    for (int w : {1, 8, 16}) run("ldsm.x4", k_ldsm, w, 2000, 1);
    for (int w : {1, 8, 16}) run("ffma x8 indep", k_ffma, w, 2000, 8);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    k_timer<<<1, 1>>>(d);
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("globaltimer min increment: %llu ns\n", h);
    return 0;
}
