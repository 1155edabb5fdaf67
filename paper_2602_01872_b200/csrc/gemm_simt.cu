// gemm_simt.cu -- CUDA-core (FFMA) implementation of the a4/a6 GEMMs.
//
// The fp32 parity path and the fallback for shapes the tcgen05 kernel (gemm_tc.cu) does not
// take.  Register-blocked 128x64 tiles, 8x4 outputs per thread, smem-staged K slices.
#include "gemm.cuh"

namespace grappa {

template <typename T> __device__ __forceinline__ float ld_f(const T* p);
template <> __device__ __forceinline__ float ld_f<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T> __device__ __forceinline__ void st_f(T* p, float v);
template <> __device__ __forceinline__ void st_f<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void st_f<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

constexpr int BM = 128, BN = 64, BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) k_gemm_nn(GemmArgs g) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int t = threadIdx.x;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int col0 = blockIdx.y * BN;
    const int tx = t & 15, ty = t >> 4;   // 16 x 16 threads: 8 rows x 4 cols each
    const int K = g.K1 + g.K2;
    const T* A1 = (const T*)g.A1;
    const T* A2 = (const T*)g.A2;
    float acc[8][4] = {};
    for (int k0 = 0; k0 < K; k0 += BK) {
        // A tile: 128 x 16 = 2048 values, 8 per thread
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int idx = t + q * 256;
            const int r = idx >> 4, kk = idx & 15;
            const int64_t gr = row0 + r;
            const int k = k0 + kk;
            float v = 0.f;
            if (gr < g.M && k < K)
                v = k < g.K1 ? ld_f<T>(A1 + gr * g.K1 + k) : ld_f<T>(A2 + gr * g.K2 + (k - g.K1));
            As[kk][r] = v;
        }
        // B tile: 16 x 64 = 1024 values, 4 per thread
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int idx = t + q * 256;
            const int kk = idx >> 6, c = idx & 63;
            const int k = k0 + kk, gc = col0 + c;
            float v = 0.f;
            if (k < K && gc < g.N) v = g.b_trans ? __ldg(g.B + (int64_t)gc * K + k) : __ldg(g.B + (int64_t)k * g.N + gc);
            Bs[kk][c] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = As[kk][ty * 8 + i];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    T* C1 = (T*)g.C1;
    T* C2 = (T*)g.C2;
    const T* mask = (const T*)g.mask;
    const int n2 = g.N - g.n_split;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int64_t r = row0 + ty * 8 + i;
        if (r >= g.M) continue;
        const float rsv = g.row_scale ? g.row_scale[r] : 1.f;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = col0 + tx * 4 + j;
            if (c >= g.N) continue;
            float v = acc[i][j];
            if (c < g.n_split) {
                v *= rsv;
                if (mask && !(ld_f<T>(mask + r * g.n_split + c) > 0.f)) v = 0.f;
                if (g.relu) v = fmaxf(v, 0.f);
                st_f<T>(C1 + r * g.n_split + c, v);
            } else {
                st_f<T>(C2 + r * n2 + (c - g.n_split), v);
            }
        }
    }
}

// dW partials: block (kt, nt, slab) computes rows [m0, m1) of [A1|A2]^T B for a 64x64 tile.
template <typename T>
__global__ void __launch_bounds__(256) k_gemm_tn(GemmTNArgs g, int64_t rows_per_slab, float* part) {
    __shared__ float As[BK][64 + 4];
    __shared__ float Bs[BK][64 + 4];
    const int t = threadIdx.x;
    const int k0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
    const int64_t m0 = (int64_t)blockIdx.z * rows_per_slab;
    const int64_t m1 = min(g.M, m0 + rows_per_slab);
    const int K = g.K1 + g.K2;
    const int tx = t & 15, ty = t >> 4;   // 4 k-rows x 4 n-cols each
    const T* A1 = (const T*)g.A1;
    const T* A2 = (const T*)g.A2;
    const T* B = (const T*)g.B;
    float acc[4][4] = {};
    for (int64_t mb = m0; mb < m1; mb += BK) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int idx = t + q * 256;
            const int mm = idx >> 6, c = idx & 63;
            const int64_t m = mb + mm;
            const int k = k0 + c, n = n0 + c;
            float va = 0.f, vb = 0.f;
            if (m < m1) {
                if (k < K) va = k < g.K1 ? ld_f<T>(A1 + m * g.K1 + k) : ld_f<T>(A2 + m * g.K2 + (k - g.K1));
                if (n < g.N) vb = ld_f<T>(B + m * g.N + n);
            }
            As[mm][c] = va;
            Bs[mm][c] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int mm = 0; mm < BK; mm++) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = As[mm][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = Bs[mm][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* P = part + (int64_t)blockIdx.z * K * g.N;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int k = k0 + ty * 4 + i;
        if (k >= K) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int n = n0 + tx * 4 + j;
            if (n < g.N) P[(int64_t)k * g.N + n] = acc[i][j];
        }
    }
}

// out[i] = sum over slabs: block = 32 outputs x 8 slab groups, group sums added in group order
// (fixed summation tree -> bitwise deterministic)
__global__ void __launch_bounds__(256) k_reduce_slabs(int64_t count, int slabs, const float* __restrict__ part,
                                                      float* __restrict__ out) {
    __shared__ float red[8][33];
    const int o = threadIdx.x & 31, gsl = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + o;
    float s = 0.f;
    if (i < count)
        for (int z = gsl; z < slabs; z += 8) s += part[(int64_t)z * count + i];
    red[gsl][o] = s;
    __syncthreads();
    if (gsl == 0 && i < count) {
        float t = 0.f;
        for (int k = 0; k < 8; k++) t += red[k][o];
        out[i] = t;
    }
}

static int slabs_for(int64_t M) {
    int64_t s = ceil_div(M, 2048);
    if (s < 1) s = 1;
    if (s > kMaxSplitK) s = kMaxSplitK;
    return (int)s;
}

size_t gemm_tn_ws_bytes(int64_t M, int K1, int K2, int N) {
    size_t simt = (size_t)slabs_for(M) * (K1 + K2) * N * sizeof(float);
    size_t tc = gemm_tc_tn_ws_bytes(M, K1, K2, N);
    return simt > tc ? simt : tc;
}

// ctx->var_gemm (grappa_set_kernel_variant "gemm"): 0 = tensor cores, 1 / 2 = CUDA-core kernels
static inline int gemm_var(const grappa_ctx* c) { return c ? c->var_gemm : 0; }

grappa_status gemm_nn(grappa_ctx* ctx, const GemmArgs& g, grappa_dtype dt, cudaStream_t s) {
    if (g.M == 0) return GRAPPA_OK;
    const double es = dt == GRAPPA_BF16 ? 2.0 : 4.0, K = g.K1 + g.K2;
    ProfScope ps(ctx, s, GRAPPA_K_GEMM,
                 (double)g.M * K * es + K * g.N * 4.0 + (double)g.M * g.N * es * (g.mask ? 2 : 1) +
                     (g.row_scale ? 4.0 * g.M : 0.0),
                 2.0 * g.M * g.N * K);
    if (dt == GRAPPA_BF16 && !gemm_var(ctx) && gemm_tc_nn_supported(g)) return gemm_tc_nn(ctx, g, s);
    if (dt == GRAPPA_F32 && !gemm_var(ctx) && gemm_x3_nn_supported(g)) return gemm_x3_nn(ctx, g, s);
    if (dt == GRAPPA_F32 && gemm_var(ctx) != 2 && sgemm_supported(g.K1, g.K2, g.N)) return sgemm_nn(ctx, g, s);
    dim3 grid((unsigned)ceil_div(g.M, BM), (unsigned)ceil_div(g.N, BN));
    if (dt == GRAPPA_BF16) k_gemm_nn<__nv_bfloat16><<<grid, 256, 0, s>>>(g);
    else k_gemm_nn<float><<<grid, 256, 0, s>>>(g);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

grappa_status gemm_tn(grappa_ctx* ctx, const GemmTNArgs& g, grappa_dtype dt, cudaStream_t s) {
    const int K = g.K1 + g.K2;
    const double es = dt == GRAPPA_BF16 ? 2.0 : 4.0;
    ProfScope ps(ctx, s, GRAPPA_K_GEMM_TN,
                 (double)g.M * K * es + (double)g.M * g.N * es + (double)K * g.N * 4.0,
                 2.0 * g.M * g.N * K);
    if (dt == GRAPPA_BF16 && !gemm_var(ctx) && g.M > 0 && gemm_tc_tn_supported(g)) return gemm_tc_tn(ctx, g, s);
    if (dt == GRAPPA_F32 && !gemm_var(ctx) && g.M > 0 && gemm_x3_tn_supported(g)) return gemm_x3_tn(ctx, g, s);
    const int slabs = g.M > 0 ? slabs_for(g.M) : 1;
    const int64_t rps = g.M > 0 ? ceil_div(g.M, slabs) : 0;
    dim3 grid((unsigned)ceil_div(K, 64), (unsigned)ceil_div(g.N, 64), (unsigned)slabs);
    if (g.M > 0) {
        if (dt == GRAPPA_F32 && gemm_var(ctx) != 2 && sgemm_supported(g.K1, g.K2, g.N)) {
            GRAPPA_TRY(sgemm_tn_partials(ctx, g, slabs, rps, s));
        } else {
            if (dt == GRAPPA_BF16) k_gemm_tn<__nv_bfloat16><<<grid, 256, 0, s>>>(g, rps, g.ws);
            else k_gemm_tn<float><<<grid, 256, 0, s>>>(g, rps, g.ws);
            GRAPPA_LAUNCHED(ctx);
        }
    } else {
        GRAPPA_CUDA(cudaMemsetAsync(g.ws, 0, (size_t)K * g.N * 4, s));
    }
    const int64_t count = (int64_t)K * g.N;
    k_reduce_slabs<<<(unsigned)ceil_div(count, 32), 256, 0, s>>>(count, g.M > 0 ? slabs : 1, g.ws, g.C);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

}  // namespace grappa
