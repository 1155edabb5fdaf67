// partition.cu -- a1: random chunking, performed once (§3.3; R1).
//
// chunk_of[v] = pi(v) mod C where pi is a seeded 4-round balanced Feistel bijection on
// [0, 2^bits) (bits = even, >= ceil(log2 N)), cycle-walked into [0, N).  Round r maps
// (L, R) -> (R, L ^ (h(seed, r, R) & mask)), h(a,b,c) = mix(a ^ mix(b ^ mix(c))), mix =
// splitmix64 finalizer.  Integer only; bit-exact with the oracle's definition.
// One thread per node; the cycle walk needs < 4 expected rounds since 2^bits < 4N.
#include "common.cuh"

namespace grappa {

__device__ __forceinline__ uint64_t dmix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_chunk_map(int64_t n, int32_t C, uint64_t seed, int half, uint64_t mask,
                            int32_t* chunk_of, unsigned long long* sizes) {
    __shared__ unsigned int cnt[64];
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        uint64_t y = (uint64_t)v;
        do {
            uint64_t L = y >> half, R = y & mask;
#pragma unroll
            for (int r = 0; r < 4; r++) {
                uint64_t nr = L ^ (dmix(seed ^ dmix((uint64_t)r ^ dmix(R))) & mask);
                L = R;
                R = nr;
            }
            y = (L << half) | R;
        } while (y >= (uint64_t)n);
        int32_t c = (int32_t)(y % (uint64_t)C);
        chunk_of[v] = c;
        if (C <= 64) atomicAdd(&cnt[c], 1u);
        else atomicAdd(&sizes[c], 1ull);
    }
    __syncthreads();
    if (C <= 64 && threadIdx.x < C && cnt[threadIdx.x])
        atomicAdd(&sizes[threadIdx.x], (unsigned long long)cnt[threadIdx.x]);
}

}  // namespace grappa

using namespace grappa;

extern "C" grappa_status grappa_partition(grappa_ctx* ctx, int64_t num_nodes, int32_t num_chunks,
                                          uint64_t seed, int32_t* chunk_of,
                                          int64_t* chunk_sizes, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && chunk_of && chunk_sizes, GRAPPA_E_ARG, "grappa_partition: null argument");
    GRAPPA_ARG(num_chunks >= 2 && (int64_t)num_chunks <= num_nodes, GRAPPA_E_ARG,
               "grappa_partition: need 2 <= C <= N (S:128-130), got C=%d N=%lld", num_chunks,
               (long long)num_nodes);
    cudaStream_t s = (cudaStream_t)stream;
    int lg = 0;
    while (((int64_t)1 << lg) < num_nodes) lg++;
    int bits = 2 * ((lg + 1) / 2);
    if (bits < 2) bits = 2;
    int half = bits / 2;
    uint64_t mask = (1ull << half) - 1;
    GRAPPA_TRY(ctx->small.grow((size_t)num_chunks * sizeof(unsigned long long)));
    unsigned long long* d_sizes = (unsigned long long*)ctx->small.p;
    GRAPPA_CUDA(cudaMemsetAsync(d_sizes, 0, (size_t)num_chunks * 8, s));
    int64_t blocks = ceil_div(num_nodes, 256);
    if (blocks > (int64_t)ctx->sm_count * 32) blocks = (int64_t)ctx->sm_count * 32;
    k_chunk_map<<<(unsigned)blocks, 256, 0, s>>>(num_nodes, num_chunks, seed, half, mask,
                                                 chunk_of, d_sizes);
    GRAPPA_LAUNCHED(ctx);
    GRAPPA_CUDA(cudaMemcpyAsync(chunk_sizes, d_sizes, (size_t)num_chunks * 8,
                                cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    // the batched repartition sizes its partitions from these counts (grappa_repartition_batch)
    ctx->cmap_ptr = chunk_of;
    ctx->cmap_n = num_nodes;
    ctx->cmap_sizes.assign(chunk_sizes, chunk_sizes + num_chunks);
    return GRAPPA_OK;
}
