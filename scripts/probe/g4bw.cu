// Row-gather throughput probe on sm_100a (L2-resident 64 MB table, 256-byte rows, random rows):
//   mode 0: TMA tile::gather4 issued by NPW warps per CTA (each lane one gather4, 32 KB per warp
//           per round, one mbarrier per warp)
//   mode 1: cp.async (LDGSTS 16 B per lane, 2 rows per warp instruction) by NPW warps, 32 KB per
//           warp per round, cp.async.mbarrier.arrive.noinc
// Prints GB/s per (mode, NPW).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0,1,0,p;}" : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int64_t n_idx, int rounds,
                  const uint4* __restrict__ table, unsigned* sink) {
    extern __shared__ __align__(1024) char buf[];
    __shared__ __align__(8) uint64_t bars[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (threadIdx.x < 32) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(&bars[threadIdx.x])), "r"(MODE == 0 ? 1 : 32));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    char* ring = buf + (size_t)w * 32768;
    const uint32_t bar = sa(&bars[w]);
    int64_t g = ((int64_t)blockIdx.x * nw + w) * 128;             // 128 rows per warp-round
    const int64_t stride = (int64_t)gridDim.x * nw * 128;
    for (int r = 0; r < rounds; r++, g += stride) {
        const int64_t base = g % (n_idx - 128);
        if (MODE == 0) {
            const int4 q = __ldg(reinterpret_cast<const int4*>(idx + base) + lane);
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(32768) : "memory");
            __syncwarp();
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(sa(ring + lane * 1024)), "l"(&tm), "r"(0), "r"(q.x), "r"(q.y), "r"(q.z), "r"(q.w), "r"(bar) : "memory");
        } else {
            const int sub = lane & 15, h = lane >> 4;
#pragma unroll 8
            for (int k2 = 0; k2 < 64; k2++) {
                const int row = __ldg(idx + base + k2 * 2 + h);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(ring + (k2 * 2 + h) * 256 + sub * 16)), "l"(table + (int64_t)row * 16 + sub) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(bar) : "memory");
        }
        wait(bar, r & 1);
    }
    if (threadIdx.x == 0 && ring[5] == 123 && ring[7] == 99) sink[0] = 1;
}
int main() {
    const int64_t rows = 64 * 1024 * 1024 / 256, n_idx = 1 << 24;
    void* fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    uint16_t* tab; cudaMalloc(&tab, rows * 256); cudaMemset(tab, 1, rows * 256);
    int* idx; cudaMalloc(&idx, n_idx * 4);
    int* h = (int*)malloc(n_idx * 4); uint64_t s = 88172645463325252ull;
    for (int64_t i = 0; i < n_idx; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % rows); }
    cudaMemcpy(idx, h, n_idx * 4, cudaMemcpyHostToDevice);
    unsigned* sink; cudaMalloc(&sink, 4);
    CUtensorMap m;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows}; cuuint64_t str[1] = {256};
    cuuint32_t box[2] = {128, 1}; cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; mode++)
        for (int npw : {1, 2, 4, 6}) {
            const int smem = npw * 32768;
            auto kern = mode == 0 ? k<0> : k<1>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int rounds = 400;
            kern<<<sms, npw * 32, smem>>>(m, idx, n_idx, 10, (const uint4*)tab, sink);
            cudaEventRecord(a);
            kern<<<sms, npw * 32, smem>>>(m, idx, n_idx, rounds, (const uint4*)tab, sink);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double bytes = (double)sms * npw * rounds * 32768.0;
            printf("mode %d (%s) warps %d: %.0f GB/s  %s\n", mode, mode ? "cp.async" : "gather4", npw, bytes / ms / 1e6, cudaGetErrorString(e));
        }
    return 0;
}
