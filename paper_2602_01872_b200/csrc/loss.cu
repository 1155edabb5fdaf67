// loss.cu -- a5: mean softmax cross-entropy over the partition's seeds + its gradient.
//
// SPEC S:276-285 (loss_and_grad), reading R8 (mean over the partition's seeds):
//   L = (1/#S) sum_{v in S} [lse(Z_v[0:K]) - Z_v[y_v]],  dZ_v = (softmax(Z_v) - e_{y_v}) / #S
// on seeds, zero on every other row and on the padded columns (masked to -inf).
// Warp per seed row; per-block partial losses in f64 combined in block order (deterministic).
#include "part.cuh"
#include "spmm.cuh"

namespace grappa {

template <typename T> __device__ __forceinline__ float lf(const T* p);
template <> __device__ __forceinline__ float lf<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float lf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T> __device__ __forceinline__ void sf(T* p, float v);
template <> __device__ __forceinline__ void sf<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void sf<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

constexpr int kLossThreads = 256;
constexpr int kMaxKPad = 512;

// seed k: logits row rows[k] (rows == null: row k), label labels[lidx ? lidx[k] : row]
template <typename T>
__global__ void __launch_bounds__(kLossThreads) k_loss(int64_t n_seeds, const int32_t* rows,
                                                       const int32_t* lidx, const int32_t* labels,
                                                       const T* logits, int K, int kpad, T* dlogits,
                                                       double* part, const float* __restrict__ rscale,
                                                       unsigned* done, double inv_n, double* out) {
    __shared__ double wsum[kLossThreads / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t k = (int64_t)blockIdx.x * (kLossThreads / 32) + wid;
    double my = 0.0;
    if (k < n_seeds) {
        const int64_t v = rows ? rows[k] : k;
        const T* z = logits + v * kpad;
        T* dz = dlogits + v * kpad;
        const int y = labels[lidx ? lidx[k] : v];
        float m = -INFINITY;
        for (int c = lane; c < K; c += 32) m = fmaxf(m, lf<T>(z + c));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float se = 0.f;
        for (int c = lane; c < K; c += 32) se += expf(lf<T>(z + c) - m);
        se = warp_sum(se);
        const float lse = m + logf(se);
        // optional row scale (GCN normalised-gradient chain, R29): dz_v * n_v
        const float inv = (1.0f / (float)n_seeds) * (rscale ? rscale[v] : 1.f);
        for (int c = lane; c < kpad; c += 32) {
            float g = 0.f;
            if (c < K) g = (expf(lf<T>(z + c) - m) / se - (c == y ? 1.f : 0.f)) * inv;
            sf<T>(dz + c, g);
        }
        if (lane == 0) my = (double)lse - (double)lf<T>(z + y);
    }
    if (lane == 0) wsum[wid] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kLossThreads / 32; w++) s += wsum[w];
        part[blockIdx.x] = s;
        // the block that completes the count combines the partials (k_loss_final's fixed order,
        // so the value is the two-launch one bit for bit) and resets the count
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int nb = (int)gridDim.x;
    const int per = (nb + 255) / 256;
    double s = 0.0;
    for (int b = threadIdx.x * per, e = min(nb, b + per); b < e; b++) s += __ldcg(part + b);
    s = warp_sum(s);
    if (lane == 0) wsum[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += wsum[w];
        *out = t * inv_n;
        *done = 0u;
    }
}

// one block: thread t sums a contiguous run of partials, then a fixed-shape tree (deterministic)
__global__ void __launch_bounds__(256) k_loss_final(int nb, const double* part, double inv_n, double* out) {
    __shared__ double ws[8];
    const int per = (nb + 255) / 256;
    double s = 0.0;
    for (int b = threadIdx.x * per, e = min(nb, b + per); b < e; b++) s += part[b];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += ws[w];
        *out = t * inv_n;
    }
}

// softmax-CE over n_seeds rows of logits [n_rows x k_pad]; dlogits fully written (zeros off
// the seed rows).  partial sums in the ctx reduction scratch (grown outside graph capture).
grappa_status loss_rows(grappa_ctx* ctx, int64_t n_seeds, const int32_t* rows, const int32_t* lidx,
                        const int32_t* labels, int64_t n_rows, const void* logits, int K, int k_pad,
                        void* dlogits, double* loss_dev, grappa_dtype dtype, cudaStream_t s,
                        const float* rscale) {
    const size_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
    ProfScope ps(ctx, s, GRAPPA_K_LOSS, (double)n_rows * k_pad * esz + 2.0 * n_seeds * k_pad * esz,
                 5.0 * n_seeds * K);
    GRAPPA_CUDA(cudaMemsetAsync(dlogits, 0, (size_t)n_rows * k_pad * esz, s));
    const int64_t nb = ceil_div(n_seeds, kLossThreads / 32);
    // the loss's own scratch: a captured epoch graph references it, and a switch prefetched on a
    // side stream (engine) may reuse the repartition workspaces while that graph runs
    // [arrival count (zero between calls) | nb partial sums]
    void* before = ctx->loss_ws.p;
    GRAPPA_TRY(ctx->loss_ws.grow((size_t)(nb + 1) * sizeof(double)));
    unsigned* done = (unsigned*)ctx->loss_ws.p;
    if (ctx->loss_ws.p != before) GRAPPA_CUDA(cudaMemsetAsync(done, 0, sizeof(double), s));
    double* part_sums = (double*)ctx->loss_ws.p + 1;
    if (n_seeds <= 0) {
        k_loss_final<<<1, 256, 0, s>>>(0, part_sums, 0.0, loss_dev);
        GRAPPA_LAUNCHED(ctx);
        return GRAPPA_OK;
    }
    const double inv_n = 1.0 / (double)n_seeds;
    if (dtype == GRAPPA_BF16)
        k_loss<__nv_bfloat16><<<(unsigned)nb, kLossThreads, 0, s>>>(
            n_seeds, rows, lidx, labels, (const __nv_bfloat16*)logits, K, k_pad, (__nv_bfloat16*)dlogits,
            part_sums, rscale, done, inv_n, loss_dev);
    else
        k_loss<float><<<(unsigned)nb, kLossThreads, 0, s>>>(n_seeds, rows, lidx, labels, (const float*)logits,
                                                            K, k_pad, (float*)dlogits, part_sums, rscale, done,
                                                            inv_n, loss_dev);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

}  // namespace grappa

using namespace grappa;

extern "C" grappa_status grappa_loss(grappa_ctx* ctx, const grappa_part* part, const void* logits,
                                     int32_t num_classes, int32_t k_pad, void* dlogits,
                                     double* loss_dev, grappa_dtype dtype, void* stream) {
    CallScope call_scope(ctx, stream);
    return grappa_loss_ex(ctx, part, logits, num_classes, k_pad, dlogits, loss_dev, dtype, 0u, stream);
}

extern "C" grappa_status grappa_loss_ex(grappa_ctx* ctx, const grappa_part* part, const void* logits,
                                        int32_t num_classes, int32_t k_pad, void* dlogits,
                                        double* loss_dev, grappa_dtype dtype, unsigned flags, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG((flags & ~GRAPPA_LOSS_DZ_NORMED) == 0, GRAPPA_E_ARG, "grappa_loss_ex: flags 0x%x invalid", flags);
    GRAPPA_ARG(ctx && part && logits && dlogits && loss_dev, GRAPPA_E_ARG, "grappa_loss: null argument");
    GRAPPA_ARG(num_classes >= 1 && num_classes <= k_pad && k_pad <= kMaxKPad, GRAPPA_E_ARG,
               "grappa_loss: need 1 <= K <= k_pad <= %d", kMaxKPad);
    const grappa_part_info& I = part->info;
    GRAPPA_ARG(I.n_seeds > 0, GRAPPA_E_EMPTY, "grappa_loss: empty seed set (S:213)");
    return loss_rows(ctx, I.n_seeds, I.seeds, nullptr, I.labels, I.n_core, logits, num_classes, k_pad,
                     dlogits, loss_dev, dtype, (cudaStream_t)stream,
                     (flags & GRAPPA_LOSS_DZ_NORMED) ? I.norm_gcn : nullptr);
}
