// gather4 semantics probe: box {W, boxrows}, which rows land where
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, const int* idx, uint16_t* out, int bytes) {
    extern __shared__ __align__(1024) char buf[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(bytes));
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :: "r"(sa(buf)), "l"(&tm), "r"(0), "r"(idx[0]), "r"(idx[1]), "r"(idx[2]), "r"(idx[3]), "r"(sa(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.b32 %0,1,0,p;}" : "=r"(done) : "r"(sa(&bar)));
    for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = ((uint16_t*)buf)[i];
}
int main() {
    const int N = 1000;
    void* fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    for (int W : {128, 48, 112, 256, 16}) for (int br : {1}) {
        std::vector<uint16_t> h((size_t)N * W);
        for (int r = 0; r < N; r++) for (int c = 0; c < W; c++) h[(size_t)r * W + c] = (uint16_t)(r * 7 + c);
        uint16_t* d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)N}; cuuint64_t str[1] = {(cuuint64_t)W * 2};
        cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)br}; cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("W=%d box rows %d: encode failed %d\n", W, br, (int)r); continue; }
        int hi[4] = {5, 999, 0, 123}; int* di; cudaMalloc(&di, 16); cudaMemcpy(di, hi, 16, cudaMemcpyHostToDevice);
        const int bytes = 4 * W * 2;
        uint16_t* dout; cudaMalloc(&dout, bytes); cudaMemset(dout, 0xff, bytes);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        k<<<1, 128, 64 * 1024>>>(m, di, dout, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint16_t> o(bytes / 2); cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int t = 0; t < 4; t++) for (int c = 0; c < W; c++) if (o[t * W + c] != (uint16_t)(hi[t] * 7 + c)) bad++;
        printf("W=%d box rows %d: %s, mismatches %d (first %u %u %u)\n", W, br, cudaGetErrorString(e), bad, o[0], o[W], o[2*W]);
        cudaFree(d); cudaFree(di); cudaFree(dout);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
