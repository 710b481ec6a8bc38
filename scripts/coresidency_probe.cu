// Probes whether two kernels' CTAs share an SM: kernel A (WA warps, ~RA registers, SA B smem) and
// kernel B (WB warps, ~RB registers, SB B smem) are launched on two streams; each CTA records
// its SM and [start, end] (globaltimer), spinning ~40 us.  Prints how many SMs hosted both at
// once.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cop scripts/coresidency_probe.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned sm() { unsigned r; asm volatile("mov.u32 %0, %smid;" : "=r"(r)); return r; }
template <int N>
__device__ void body(unsigned long long* rec, float seed) {
    extern __shared__ float s[];
    float acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = seed * (i + 1);
    unsigned long long t0 = gt();
    while (gt() - t0 < 40000) {
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = acc[i] * 1.0001f + (float)i;
    }
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) sum += acc[i];
    if (sum == 12345.f) s[threadIdx.x] = sum;
    if (threadIdx.x == 0) { rec[blockIdx.x * 3] = sm(); rec[blockIdx.x * 3 + 1] = t0; rec[blockIdx.x * 3 + 2] = gt(); }
}
template <int N> __global__ void ka(unsigned long long* r, float x) { body<N>(r, x); }
template <int N> __global__ void kb(unsigned long long* r, float x) { body<N>(r, x); }

template <int NA, int NB>
void run(int wa, int sa, int wb, int sb) {
    cudaFuncSetAttribute(ka<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(kb<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(ka<NA>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(kb<NB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncAttributes fa, fb;
    cudaFuncGetAttributes(&fa, ka<NA>);
    cudaFuncGetAttributes(&fb, kb<NB>);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *ra, *rb;
    cudaMalloc(&ra, nsm * 24);
    cudaMalloc(&rb, nsm * 24);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    ka<NA><<<nsm, wa * 32, sa, s1>>>(ra, 1.f);
    kb<NB><<<nsm, wb * 32, sb, s2>>>(rb, 2.f);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> ha(nsm * 3), hb(nsm * 3);
    cudaMemcpy(ha.data(), ra, nsm * 24, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), rb, nsm * 24, cudaMemcpyDeviceToHost);
    int both = 0;
    for (int i = 0; i < nsm; ++i)
        for (int j = 0; j < nsm; ++j)
            if (ha[i * 3] == hb[j * 3] && ha[i * 3 + 1] < hb[j * 3 + 2] && hb[j * 3 + 1] < ha[i * 3 + 2]) { ++both; break; }
    printf("A: %2d warps %3d regs %6d smem | B: %2d warps %3d regs %6d smem | regs/SM %6d | SMs with A and B overlapping: %d  (%s)\n",
           wa, fa.numRegs, sa, wb, fb.numRegs, sb, wa * 32 * fa.numRegs + wb * 32 * fb.numRegs, both,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(ra); cudaFree(rb);
}
int main() {
    run<72, 112>(9, 115728, 10, 112256);   // the ring pair v2 shapes (~80 / ~120 regs)
    run<72, 112>(9, 60000, 10, 60000);     // same registers, small smem
    run<72, 112>(8, 60000, 8, 60000);      // 8-warp CTAs
    run<72, 112>(8, 115728, 8, 112256);
    run<40, 80>(9, 60000, 10, 60000);      // fewer registers
    run<24, 60>(9, 60000, 10, 60000);
    run<72, 112>(12, 60000, 8, 60000);
    run<24, 24>(9, 115728, 10, 112256);    // smem only
    run<24, 24>(9, 107000, 10, 109000);
    return 0;
}
