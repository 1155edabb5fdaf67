// gemm_f32.cu -- fp32 CUDA-core GEMMs for the fp32-storage (1e-4 parity) path.
//
// fp32 storage normally runs on the split-fp32 tcgen05 kernels (gemm_tc.cu: bf16 hi + lo
// operands, 3 MMAs per K step; plain TF32 rounds operands to 10 mantissa bits and misses the
// 1e-4 bar).  These FFMA kernels serve the shapes those do not take and the cross-check
// variant (grappa_set_kernel_variant("gemm", 1)): 128x128 tiles, 8x8 outputs per thread in two 4x4
// quadrants (conflict-free float4 smem reads), 8-deep K slices double-buffered through shared
// memory with the next slice prefetched into registers.
//   k_sgemm_nn : C = [A1 | A2] * op(B)  (+ row-scale / relu'-mask / ReLU epilogue, column split)
//   k_sgemm_tn : fp32 partials of [A1 | A2]^T * Bm over a row slab (weight gradient)
#include "gemm.cuh"

namespace grappa {

constexpr int SM_ = 128, SN_ = 128, SK_ = 8;

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__global__ void __launch_bounds__(256, 2) k_sgemm_nn(GemmArgs g) {
    __shared__ __align__(16) float As[2][SK_][SM_];
    __shared__ __align__(16) float Bs[2][SK_][SN_];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * SM_;
    const int col0 = blockIdx.y * SN_;
    const int K = g.K1 + g.K2;
    const float* A1 = (const float*)g.A1;
    const float* A2 = (const float*)g.A2;
    // this thread's global-load coordinates
    const int ar = t >> 1, ak = (t & 1) * 4;               // A: row, k offset (4 wide)
    const int bk = t >> 5, bn = (t & 31) * 4;              // B (normal): k row, n offset
    const int tn = t >> 1, tk = (t & 1) * 4;               // B (trans): n, k offset
    auto load_a = [&](int k0) -> float4 {
        const int64_t r = row0 + ar;
        const int k = k0 + ak;
        if (r >= g.M || k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
        return k < g.K1 ? ld4(A1 + r * g.K1 + k) : ld4(A2 + r * g.K2 + (k - g.K1));
    };
    auto load_b = [&](int k0) -> float4 {
        if (!g.b_trans) {
            const int k = k0 + bk, n = col0 + bn;
            if (k >= K || n >= g.N) return make_float4(0.f, 0.f, 0.f, 0.f);
            return ld4(g.B + (int64_t)k * g.N + n);
        }
        const int n = col0 + tn, k = k0 + tk;
        if (n >= g.N || k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
        return ld4(g.B + (int64_t)n * K + k);
    };
    auto store = [&](int buf, float4 a, float4 b) {
        As[buf][ak + 0][ar] = a.x; As[buf][ak + 1][ar] = a.y; As[buf][ak + 2][ar] = a.z; As[buf][ak + 3][ar] = a.w;
        if (!g.b_trans) {
            *reinterpret_cast<float4*>(&Bs[buf][bk][bn]) = b;
        } else {
            Bs[buf][tk + 0][tn] = b.x; Bs[buf][tk + 1][tn] = b.y; Bs[buf][tk + 2][tn] = b.z; Bs[buf][tk + 3][tn] = b.w;
        }
    };
    float acc[8][8] = {};
    float4 ra = load_a(0), rb = load_b(0);
    store(0, ra, rb);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += SK_) {
        const bool more = k0 + SK_ < K;
        if (more) { ra = load_a(k0 + SK_); rb = load_b(k0 + SK_); }
#pragma unroll
        for (int kk = 0; kk < SK_; kk++) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store(buf ^ 1, ra, rb);
            __syncthreads();
            buf ^= 1;
        }
    }
    float* C1 = (float*)g.C1;
    float* C2 = (float*)g.C2;
    const float* mask = (const float*)g.mask;
    const int n2 = g.N - g.n_split;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int64_t r = row0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (r >= g.M) continue;
        const float rsv = g.row_scale ? g.row_scale[r] : 1.f;
#pragma unroll
        for (int jh = 0; jh < 2; jh++) {
            const int c = col0 + jh * 64 + tx * 4;       // 4 consecutive columns
            if (c >= g.N) continue;
            float v[4] = {acc[i][jh * 4], acc[i][jh * 4 + 1], acc[i][jh * 4 + 2], acc[i][jh * 4 + 3]};
            if (c < g.n_split) {
#pragma unroll
                for (int q = 0; q < 4; q++) v[q] *= rsv;
                if (mask) {
                    const float4 m = ld4(mask + r * g.n_split + c);
                    v[0] = m.x > 0.f ? v[0] : 0.f; v[1] = m.y > 0.f ? v[1] : 0.f;
                    v[2] = m.z > 0.f ? v[2] : 0.f; v[3] = m.w > 0.f ? v[3] : 0.f;
                }
                if (g.relu) {
#pragma unroll
                    for (int q = 0; q < 4; q++) v[q] = fmaxf(v[q], 0.f);
                }
                *reinterpret_cast<float4*>(C1 + r * g.n_split + c) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
                *reinterpret_cast<float4*>(C2 + r * n2 + (c - g.n_split)) = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    }
}

// partial[slab][k][n] = sum_{rows of the slab} [A1|A2][row][k] * B[row][n] for a 128x128 tile
__global__ void __launch_bounds__(256) k_sgemm_tn(GemmTNArgs g, int64_t rows_per_slab, float* part) {
    __shared__ __align__(16) float As[2][SK_][SM_];
    __shared__ __align__(16) float Bs[2][SK_][SN_];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int k0 = blockIdx.x * SM_, n0 = blockIdx.y * SN_;
    const int64_t m0 = (int64_t)blockIdx.z * rows_per_slab;
    const int64_t m1 = min(g.M, m0 + rows_per_slab);
    const int K = g.K1 + g.K2;
    const float* A1 = (const float*)g.A1;
    const float* A2 = (const float*)g.A2;
    const float* B = (const float*)g.B;
    const int lr = t >> 5, lc = (t & 31) * 4;              // 8 rows x 32 float4
    auto load_a = [&](int64_t mb) -> float4 {
        const int64_t m = mb + lr;
        const int k = k0 + lc;
        if (m >= m1 || k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
        return k < g.K1 ? ld4(A1 + m * g.K1 + k) : ld4(A2 + m * g.K2 + (k - g.K1));
    };
    auto load_b = [&](int64_t mb) -> float4 {
        const int64_t m = mb + lr;
        const int n = n0 + lc;
        if (m >= m1 || n >= g.N) return make_float4(0.f, 0.f, 0.f, 0.f);
        return ld4(B + m * g.N + n);
    };
    float acc[8][8] = {};
    float4 ra = load_a(m0), rb = load_b(m0);
    *reinterpret_cast<float4*>(&As[0][lr][lc]) = ra;
    *reinterpret_cast<float4*>(&Bs[0][lr][lc]) = rb;
    __syncthreads();
    int buf = 0;
    for (int64_t mb = m0; mb < m1; mb += SK_) {
        const bool more = mb + SK_ < m1;
        if (more) { ra = load_a(mb + SK_); rb = load_b(mb + SK_); }
#pragma unroll
        for (int kk = 0; kk < SK_; kk++) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            *reinterpret_cast<float4*>(&As[buf ^ 1][lr][lc]) = ra;
            *reinterpret_cast<float4*>(&Bs[buf ^ 1][lr][lc]) = rb;
            __syncthreads();
            buf ^= 1;
        }
    }
    float* P = part + (int64_t)blockIdx.z * K * g.N;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int k = k0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (k >= K) continue;
#pragma unroll
        for (int jh = 0; jh < 2; jh++) {
            const int n = n0 + jh * 64 + tx * 4;
            if (n >= g.N) continue;
            *reinterpret_cast<float4*>(P + (int64_t)k * g.N + n) =
                make_float4(acc[i][jh * 4], acc[i][jh * 4 + 1], acc[i][jh * 4 + 2], acc[i][jh * 4 + 3]);
        }
    }
}

bool sgemm_supported(int K1, int K2, int N) { return K1 % 4 == 0 && K2 % 4 == 0 && N % 4 == 0; }

grappa_status sgemm_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(g.M, SM_), (unsigned)ceil_div(g.N, SN_));
    k_sgemm_nn<<<grid, 256, 0, s>>>(g);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

grappa_status sgemm_tn_partials(grappa_ctx* ctx, const GemmTNArgs& g, int slabs, int64_t rps, cudaStream_t s) {
    const int K = g.K1 + g.K2;
    dim3 grid((unsigned)ceil_div(K, SM_), (unsigned)ceil_div(g.N, SN_), (unsigned)slabs);
    k_sgemm_tn<<<grid, 256, 0, s>>>(g, rps, g.ws);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

}  // namespace grappa
