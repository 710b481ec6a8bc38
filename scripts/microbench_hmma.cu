// mma.sync.m16n8k16 bf16 throughput / latency on sm_100a (legacy warp-level MMA on a tcgen05 part).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbh scripts/microbench_hmma.cu && /tmp/mbh
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CH>   // CH independent accumulator chains per warp
__global__ void k(float* out, long long* cyc, int iters) {
    float d[CH][4] = {};
    uint32_t a = threadIdx.x, b = threadIdx.x * 3;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) mma(d[c], a, a + 1, a + 2, a + 3, b, b + c);
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8 * 148);
    const int it = 1000;
    k<CH><<<1, warps * 32>>>(o, c, it);
    k<CH><<<1, warps * 32>>>(o, c, it);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d chains %d: %.1f cycles per MMA per warp, %.2f MMA/cycle/SM\n", warps, CH, (double)h / (it * CH),
           (double)warps * it * CH / h);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<1>(1); run<4>(1); run<8>(1);
    run<1>(4); run<4>(4); run<8>(4);
    run<1>(8); run<4>(8); run<8>(8);
    run<4>(16); run<8>(16);
    return 0;
}
