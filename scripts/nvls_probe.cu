// NVLS multicast probe: can this process create a multicast object on its GPU, bind memory, map it and
// run multimem.ld_reduce / multimem.red over it (world 1)?  nvcc -gencode arch=compute_100a,code=sm_100a
// -o /tmp/nvls scripts/nvls_probe.cu -lcuda && /tmp/nvls
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("%s -> %d %s\n", #x, (int)r_, s_); return 1; } } while (0)
__global__ void k(float* mc, float* uc, float* out, unsigned* mflag, unsigned* uflag) {
    int i = threadIdx.x;
    uc[i] = 1.5f * i;
    __threadfence_system();
    __syncthreads();
    if (i == 0) asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mflag), "r"(1u) : "memory");
    if (i == 0) { unsigned v; do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(uflag)); } while (v < 1); }
    __syncthreads();
    float s;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(s) : "l"(mc + i) : "memory");
    out[i] = s;
}
int main() {
    CK(cuInit(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("MULTICAST_SUPPORTED = %d\n", mcs);
    cudaSetDevice(0); cudaFree(0);
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1; mp.size = 2 << 20; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("granularity %zu\n", gran);
    mp.size = ((mp.size + gran - 1) / gran) * gran;
    CUmemGenericAllocationHandle mch;
    {
        const unsigned long long hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_FABRIC};
        bool ok = false;
        for (int nd = 1; nd <= 2 && !ok; ++nd)
            for (int h = 0; h < 3 && !ok; ++h) {
                CUmulticastObjectProp q = mp; q.numDevices = nd; q.handleTypes = hts[h];
                CUresult r = cuMulticastCreate(&mch, &q);
                printf("cuMulticastCreate(numDevices=%d, handleTypes=%llu) -> %d\n", nd, hts[h], (int)r);
                if (r == CUDA_SUCCESS && nd == 1) { ok = true; mp = q; }
            }
        if (!ok) return 1;
    }
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, mp.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
    CUdeviceptr uva, mva;
    CK(cuMemAddressReserve(&uva, mp.size, gran, 0, 0)); CK(cuMemMap(uva, mp.size, 0, ph, 0));
    CK(cuMemAddressReserve(&mva, mp.size, gran, 0, 0)); CK(cuMemMap(mva, mp.size, 0, mch, 0));
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, mp.size, &ad, 1)); CK(cuMemSetAccess(mva, mp.size, &ad, 1));
    cudaMemset((void*)uva, 0, mp.size);
    float* out; cudaMalloc(&out, 256 * 4);
    k<<<1, 64>>>((float*)mva, (float*)uva, out, (unsigned*)(mva + (1 << 20)), (unsigned*)(uva + (1 << 20)));
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    float h[64]; cudaMemcpy(h, out, 256, cudaMemcpyDeviceToHost);
    printf("out[3] = %f (want 4.5), out[63] = %f (want 94.5)\n", h[3], h[63]);
    return 0;
}
