// Probes the per-SM shared-memory accounting on this GPU: for a kernel of 288 threads and dynamic
// SMEM X, how many CTAs fit one SM (cudaOccupancyMaxActiveBlocksPerMultiprocessor), and the
// dynamic SMEM available per CTA when n CTAs share an SM.  nvcc -arch=sm_100a scripts/smem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    printf("smemPerSM %zu smemPerBlockOptin %zu reservedPerBlock %zu regsPerSM %d\n", pr.sharedMemPerMultiprocessor,
           pr.sharedMemPerBlockOptin, pr.reservedSharedMemPerBlock, pr.regsPerMultiprocessor);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (int n = 1; n <= 4; ++n) {
        size_t dyn = 0;
        cudaOccupancyAvailableDynamicSMemPerBlock(&dyn, k, n, 288);
        printf("blocks/SM %d -> available dynamic smem per block %zu\n", n, dyn);
    }
    int prev = -1;
    for (int x = 100 * 1024; x <= 120 * 1024; x += 128) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 288, x);
        if (nb != prev) { printf("dyn smem %d -> %d blocks/SM\n", x, nb); prev = nb; }
    }
    return 0;
}
