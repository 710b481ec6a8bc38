// Probe of TMA tile::gather4 semantics on sm_100a: which tensor-map box height works and
// what smem layout results (SWIZZLE_128B).  build:
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/g4 scripts/test_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_gather(const __grid_constant__ CUtensorMap tm, int4 rows, int col, uint16_t* out, int nbytes) {
    __shared__ __align__(1024) uint16_t buf[4 * 64 * 2];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4 * 64 * 2; ++i) buf[i] = 0xFFFF;
        uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(buf)),
            "l"(&tm), "r"(col), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w), "r"(b)
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b));
        for (int i = 0; i < 4 * 64 * 2; ++i) out[i] = buf[i];
    }
}

int main() {
    const int R = 64, C = 128;
    std::vector<uint16_t> h(R * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
    uint16_t *d, *dout;
    cudaMalloc(&d, R * C * 2);
    cudaMalloc(&dout, 4 * 64 * 2 * 2);
    cudaMemcpy(d, h.data(), R * C * 2, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int bh : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
        cuuint64_t strides[1] = {(cuuint64_t)C * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)bh};
        cuuint32_t es[2] = {1, 1};
        CUresult res = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box height %d: encode %d\n", bh, (int)res);
        if (res != CUDA_SUCCESS) continue;
        cudaMemset(dout, 0, 4 * 64 * 2 * 2);
        k_gather<<<1, 32>>>(tm, make_int4(5, 17, 2, 40), 64, dout, 4 * 64 * 2);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  kernel: %s\n", cudaGetErrorString(e));
        if (e != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        std::vector<uint16_t> o(4 * 64 * 2);
        cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
        for (int row = 0; row < 5; ++row) {
            printf("  smem row %d:", row);
            for (int c = 0; c < 64; c += 8) printf(" %04x", o[row * 64 + c]);
            printf("\n");
        }
    }
    return 0;
}
