// load_kernel.cu -- cold-start copy of one adapter's rank rows (§2.3 C1) as a
// zero-copy gather kernel: the SMs read the pinned, UVA-mapped host rows over PCIe with 16-B loads
// and write them to the adapter's pool pages (LORA_OPT_LOAD_KERNEL; default: cudaMemcpyAsync per
// run of consecutive pages).  Many SMs keep many PCIe reads in flight, where a DMA engine pays a
// setup cost per sub-MB copy.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernel_config.h"
#include "plan.h"

namespace lora {

struct LoadArgs {
    char* dA;
    char* dB;
    const char* sA;   // device-visible address of the pinned host rows [rank][H_in]
    const char* sB;
    int64_t ra, rb;   // row bytes
    int rank;
    int32_t pages[LORA_MAX_RANK];
};

__global__ void __launch_bounds__(256) lora_load_kernel(const __grid_constant__ LoadArgs a) {
    const int64_t va = a.ra / 16, vb = a.rb / 16;
    const int64_t total = (int64_t)a.rank * (va + vb);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t per = va + vb;
        const int j = (int)(i / per);
        const int64_t q = i - (int64_t)j * per;
        uint4 v;
        char* dst;
        const char* src;
        if (q < va) {
            src = a.sA + j * a.ra + q * 16;
            dst = a.dA + (int64_t)a.pages[j] * a.ra + q * 16;
        } else {
            src = a.sB + j * a.rb + (q - va) * 16;
            dst = a.dB + (int64_t)a.pages[j] * a.rb + (q - va) * 16;
        }
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src));
        *reinterpret_cast<uint4*>(dst) = v;
    }
}

int launch_load(char* dA, char* dB, const void* sA, const void* sB, int64_t ra, int64_t rb, int rank,
                const int32_t* pages, int num_sms, lora_cuda_stream st) {
    LoadArgs a;
    a.dA = dA;
    a.dB = dB;
    a.sA = static_cast<const char*>(sA);
    a.sB = static_cast<const char*>(sB);
    a.ra = ra;
    a.rb = rb;
    a.rank = rank;
    for (int j = 0; j < rank; ++j) a.pages[j] = pages[j];
    const int64_t work = (int64_t)rank * ((ra + rb) / 16);
    int grid = (int)((work + 255) / 256);
    if (grid > 2 * num_sms) grid = 2 * num_sms;
    lora_load_kernel<<<grid, 256, 0, st>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace lora
