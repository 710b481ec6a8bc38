// Max active clusters of a 256-thread kernel vs cluster size and dynamic smem (B200 GPC packing).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cocc scripts/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ char s[]; if (p) p[0] = s[0]; }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int smems[] = {40, 56, 72, 84, 100, 110, 150, 200};
    for (int cl : {1, 2, 4, 8, 16}) {
        for (int kb : smems) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cl * 64);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = kb * 1024;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
            printf("cluster %2d smem %3d KB: max active clusters %4d (CTAs %4d) %s\n", cl, kb, n, n * cl,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
}
