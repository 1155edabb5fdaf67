// gat.cu -- GAT layers on the isolated local CSR (reading R35: one
// head, self loop, LeakyReLU 0.2, no bias).
//
//   z = h W (GEMM),  s = h (W a_src),  t = h (W a_dst)  (fp32, k_gat_st: one pass over h)
//   alpha_vu = exp(lrelu(s_u + t_v) - lse_v),  u in N_loc(v) + v  (k_gat_alpha, warp per row)
//   Z_v = sum_u alpha_vu z_u                                    (the SpMM, per-edge weights)
// backward, given g = dL/dZ:
//   d_vu = g_v . z_u,  c_v = sum_u alpha_vu d_vu,  lam = lrelu'(s_u + t_v)
//   dt_v = sum_u alpha_vu (d_vu - c_v) lam                       (k_gat_rows: forward rows)
//   dz_u = sum_v alpha_vu g_v + ds_u a_src + dt_u a_dst,
//   ds_u = sum_v alpha_vu (d_vu - c_v) lam                       (k_gat_cols: transpose rows)
//   dW = h^T dz,  [da_src da_dst] = z^T [ds dt],  dh = dz W^T    (the GEMMs)
// All sums run in a fixed order (no atomics): bitwise reproducible.
#include "gemm.cuh"
#include "part.cuh"
#include "spmm.cuh"

namespace grappa {

constexpr float kSlope = 0.2f;     // LeakyReLU negative slope (R35)
constexpr int kHW = 32;            // warps per block of the block-per-hub-row kernels

template <typename T> struct GV;
template <> struct GV<float> {
    static constexpr int E = 4;
    __device__ static void load(const float* p, float* f) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    }
    __device__ static void store(float* p, const float* f) {
        *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    }
    __device__ static float get(const float* p) { return __ldg(p); }
};
template <> struct GV<__nv_bfloat16> {
    static constexpr int E = 8;
    __device__ static void load(const __nv_bfloat16* p, float* f) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    __device__ static void store(__nv_bfloat16* p, const float* f) {
        uint4 v;
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&b);
        }
        *reinterpret_cast<uint4*>(p) = v;
    }
    __device__ static float get(const __nv_bfloat16* p) { return __bfloat162float(*p); }
};

__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : kSlope * x; }
__device__ __forceinline__ float lrelu_d(float x) { return x > 0.f ? 1.f : kSlope; }

// wa = [W a_src; W a_dst]  (2 x K fp32), w = [W; a_src; a_dst]  (s = h (W a_src) = (h W) a_src)
__global__ void k_gat_wa(int K, int N, const float* __restrict__ w, float* __restrict__ wa) {
    const float* as = w + (int64_t)K * N;
    const float* ad = as + N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * K; i += gridDim.x * blockDim.x) {
        const int k = i % K;
        const float* a = i < K ? as : ad;
        float v = 0.f;
        for (int c = 0; c < N; c++) v = fmaf(w[(int64_t)k * N + c], a[c], v);
        wa[i] = v;
    }
}

// s_v, t_v in fp32 straight from h_in (one pass over h_in; a bf16-rounded z would cost the
// attention logits their precision): warp per row, lanes over 16-byte vectors of the row
template <typename T>
__global__ void k_gat_st(int64_t n, int K, const T* __restrict__ h, const float* __restrict__ wa,
                         float4* __restrict__ att) {
    constexpr int E = GV<T>::E;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nv = K / E;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nwarps) {
        float ps = 0.f, pt = 0.f;
        for (int c = lane; c < nv; c += 32) {
            float f[E];
            GV<T>::load(h + v * K + c * E, f);
#pragma unroll
            for (int q = 0; q < E; q++) {
                ps = fmaf(f[q], wa[c * E + q], ps);
                pt = fmaf(f[q], wa[K + c * E + q], pt);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ps += __shfl_xor_sync(0xffffffffu, ps, o);
            pt += __shfl_xor_sync(0xffffffffu, pt, o);
        }
        if (lane == 0) att[v] = make_float4(ps, pt, 0.f, 0.f);
    }
}

// warp per row: lse over N(v) + v, alpha per edge (CSR order) and for the self loop;
// att[v] = {s_v, t_v, lse_v, .}
__global__ void k_gat_alpha(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            float* __restrict__ alpha, float* __restrict__ alpha_self, float4* __restrict__ att) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nwarps) {
        const int64_t e0 = rowptr[v], e1 = rowptr[v + 1];
        if (e1 - e0 > kSegLen) continue;                 // hub rows: k_gat_alpha_heavy
        const float4 av = att[v];
        const float sv = av.x, tv = av.y;
        const float eself = lrelu(sv + tv);
        // online max / sum per lane, then a fixed-order warp combine
        float m = lane == 0 ? eself : -INFINITY, sum = lane == 0 ? 1.f : 0.f;
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            const float x = lrelu(att[col[e]].x + tv);
            if (x > m) { sum = sum * __expf(m - x) + 1.f; m = x; }
            else sum += __expf(x - m);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
            const float mm = fmaxf(m, m2);
            sum = (m == -INFINITY ? 0.f : sum * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
            m = mm;
        }
        const float lse = m + __logf(sum);
        for (int64_t e = e0 + lane; e < e1; e += 32) alpha[e] = __expf(lrelu(att[col[e]].x + tv) - lse);
        if (lane == 0) {
            alpha_self[v] = __expf(eself - lse);
            att[v].z = lse;
        }
    }
}

// hub rows (deg > kSegLen), one kHW-warp block each: per-thread online (max, sum), combined
// across lanes then warps in a fixed order; then every thread writes its edges' coefficients
__global__ void __launch_bounds__(kHW * 32) k_gat_alpha_heavy(const int32_t* __restrict__ heavy_rows,
                                                               const int64_t* __restrict__ rowptr,
                                                               const int32_t* __restrict__ col,
                                                               float* __restrict__ alpha, float* __restrict__ alpha_self,
                                                               float4* __restrict__ att) {
    __shared__ float sm[kHW], ss[kHW];
    __shared__ float s_lse;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t v = heavy_rows[blockIdx.x];
    const int64_t e0 = rowptr[v], e1 = rowptr[v + 1];
    const float4 av = att[v];
    const float tv = av.y, eself = lrelu(av.x + av.y);
    float m = threadIdx.x == 0 ? eself : -INFINITY, sum = threadIdx.x == 0 ? 1.f : 0.f;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const float x = lrelu(att[col[e]].x + tv);
        if (x > m) { sum = sum * __expf(m - x) + 1.f; m = x; }
        else sum += __expf(x - m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        const float mm = fmaxf(m, m2);
        sum = (m == -INFINITY ? 0.f : sum * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
        m = mm;
    }
    if (lane == 0) { sm[w] = m; ss[w] = sum; }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.f;
        for (int k = 0; k < kHW; k++) {
            const float mm = fmaxf(M, sm[k]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - mm)) + (sm[k] == -INFINITY ? 0.f : ss[k] * __expf(sm[k] - mm));
            M = mm;
        }
        s_lse = M + __logf(S);
        alpha_self[v] = __expf(eself - s_lse);
        att[v].z = s_lse;
    }
    __syncthreads();
    const float lse = s_lse;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) alpha[e] = __expf(lrelu(att[col[e]].x + tv) - lse);
}

// induced-core: the CSR is symmetric with ascending rows, so the transpose is the CSR itself and
// the forward edge of transposed entry e (row u, neighbour v = col[e]) is (v -> u): found by
// binary search in row v
__global__ void k_gat_rev(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                          int32_t* __restrict__ rev) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        for (int64_t e = rowptr[u] + lane; e < rowptr[u + 1]; e += 32) {
            const int32_t v = col[e];
            int64_t lo = rowptr[v], hi = rowptr[v + 1] - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col[mid] < u) lo = mid + 1; else hi = mid;
            }
            rev[e] = (int32_t)lo;
        }
    }
}

// Per-row statistics of the backward (forward rows): c_v = sum alpha d, dt_v = sum alpha (d - c) lam
// computed as A = sum alpha d, B = sum alpha d lam, C = sum alpha lam -> dt = B - A C.
// Group of G2 lanes per row (G = width / EPV active lanes with one 16-byte vector each).
// Light rows (deg <= kSegLen) here; heavy rows by k_gat_rows_heavy.
struct RowAcc { float A, B, C; };

template <typename T>
__device__ __forceinline__ float group_sum(float x, int G2) {
    for (int o = G2 >> 1; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

template <typename T>
__global__ void __launch_bounds__(256) k_gat_rows(int64_t n, const int4* __restrict__ desc, const int32_t* __restrict__ col,
                                                  const T* __restrict__ z, const T* __restrict__ g,
                                                  const float* __restrict__ alpha, const float* __restrict__ alpha_self,
                                                  float4* __restrict__ att, float* __restrict__ dt, int W, int G, int G2) {
    constexpr int E = GV<T>::E;
    const int lane = threadIdx.x & 31;
    const int P = 32 / G2, slot = lane / G2, sub = lane % G2;
    const int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * P;
    const int64_t ri = base + slot;
    int64_t v = -1, e0 = 0, e1 = 0;
    if (ri < n) {
        const int4 d = __ldg(desc + ri);
        if (d.y <= kSegLen) {
            v = d.x;
            e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
            e1 = e0 + d.y;
        }
    }
    // uniform trip count across the warp
    int64_t len = e1 - e0;
    int64_t mx = len;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
    float gv[E];
    float tv = 0.f;
#pragma unroll
    for (int q = 0; q < E; q++) gv[q] = 0.f;
    if (v >= 0) {
        if (sub < G) GV<T>::load(g + v * W + sub * E, gv);
        tv = att[v].y;
    }
    RowAcc r{0.f, 0.f, 0.f};
    for (int64_t k = 0; k < mx; k++) {
        const bool ok = k < len;
        const int32_t u = ok ? col[e0 + k] : 0;
        float p = 0.f;
        if (ok && sub < G) {
            float zu[E];
            GV<T>::load(z + (int64_t)u * W + sub * E, zu);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gv[q], zu[q], p);
        }
        const float dd = group_sum<T>(p, G2);
        if (ok) {
            const float a = alpha[e0 + k], lam = lrelu_d(att[u].x + tv);
            r.A = fmaf(a, dd, r.A);
            r.B = fmaf(a * dd, lam, r.B);
            r.C = fmaf(a, lam, r.C);
        }
    }
    // self loop, last
    float p = 0.f;
    if (v >= 0 && sub < G) {
        float zv[E];
        GV<T>::load(z + v * W + sub * E, zv);
#pragma unroll
        for (int q = 0; q < E; q++) p = fmaf(gv[q], zv[q], p);
    }
    const float dd = group_sum<T>(p, G2);
    if (v >= 0 && sub == 0) {
        const float4 av = att[v];
        const float a = alpha_self[v], lam = lrelu_d(av.x + av.y);
        r.A = fmaf(a, dd, r.A);
        r.B = fmaf(a * dd, lam, r.B);
        r.C = fmaf(a, lam, r.C);
        att[v].w = r.A;
        dt[v] = r.B - r.A * r.C;
    }
}

// heavy rows (deg > kSegLen): one kHW-warp block per row; warp w takes the contiguous edge range
// [w L/kHW, (w+1) L/kHW), its P lane groups every P-th edge of it; group sums are combined in slot
// order, warp sums in warp order, the self loop last (deterministic).
template <typename T>
__global__ void __launch_bounds__(kHW * 32) k_gat_rows_heavy(const int32_t* __restrict__ heavy_rows,
                                                        const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                        const T* __restrict__ z, const T* __restrict__ g,
                                                        const float* __restrict__ alpha, const float* __restrict__ alpha_self,
                                                        float4* __restrict__ att, float* __restrict__ dt, int W, int G, int G2) {
    constexpr int E = GV<T>::E;
    __shared__ RowAcc part[kHW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t v = heavy_rows[blockIdx.x];
    const int64_t r0 = rowptr[v], r1 = rowptr[v + 1], L = r1 - r0;
    // the warp's lanes: P = 32/G2 groups, each takes every P-th edge of the warp's range
    const int P = 32 / G2, slot = lane / G2, sub = lane % G2;
    const int64_t w0 = r0 + L * w / kHW, w1 = r0 + L * (w + 1) / kHW;
    float gv[E];
    const float tv = att[v].y;
    if (sub < G) GV<T>::load(g + v * W + sub * E, gv);
    else {
#pragma unroll
        for (int q = 0; q < E; q++) gv[q] = 0.f;
    }
    RowAcc r{0.f, 0.f, 0.f};
    const int64_t trips = (w1 - w0 + P - 1) / P;
    for (int64_t k = 0; k < trips; k++) {
        const int64_t e = w0 + k * P + slot;
        const bool ok = e < w1;
        const int32_t u = ok ? col[e] : 0;
        float p = 0.f;
        if (ok && sub < G) {
            float zu[E];
            GV<T>::load(z + (int64_t)u * W + sub * E, zu);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gv[q], zu[q], p);
        }
        const float dd = group_sum<T>(p, G2);
        if (ok) {
            const float a = alpha[e], lam = lrelu_d(att[u].x + tv);
            r.A = fmaf(a, dd, r.A);
            r.B = fmaf(a * dd, lam, r.B);
            r.C = fmaf(a, lam, r.C);
        }
    }
    // combine the P groups of the warp (sub == 0 lanes hold each group's sums), in slot order
    RowAcc t{0.f, 0.f, 0.f};
    for (int k = 0; k < P; k++) {
        const float A = __shfl_sync(0xffffffffu, r.A, k * G2), B = __shfl_sync(0xffffffffu, r.B, k * G2),
                    C = __shfl_sync(0xffffffffu, r.C, k * G2);
        t.A += A; t.B += B; t.C += C;
    }
    if (lane == 0) part[w] = t;
    __syncthreads();
    // self loop (warp 0), then the fixed-order combine
    if (w == 0) {
        float p = 0.f;
        if (sub < G && slot == 0) {
            float zv[E];
            GV<T>::load(z + v * W + sub * E, zv);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gv[q], zv[q], p);
        }
        const float dd = group_sum<T>(p, G2);
        if (lane == 0) {
            RowAcc s{0.f, 0.f, 0.f};
            for (int k = 0; k < kHW; k++) { s.A += part[k].A; s.B += part[k].B; s.C += part[k].C; }
            const float4 av = att[v];
            const float a = alpha_self[v], lam = lrelu_d(av.x + av.y);
            s.A = fmaf(a, dd, s.A);
            s.B = fmaf(a * dd, lam, s.B);
            s.C = fmaf(a, lam, s.C);
            att[v].w = s.A;
            dt[v] = s.B - s.A * s.C;
        }
    }
}

// Transpose rows u: dz_u = sum_v alpha_vu g_v (+ alpha_uu g_u) + ds_u a_src + dt_u a_dst,
// ds_u = sum_v alpha_vu (g_v . z_u - c_v) lam_vu (+ self).  alpha_vu = alpha[eid[e]].
// Writes dz [n x W] (dtype) and DS [n x 16] = {ds, dt, 0...} (dtype).
template <typename T>
__device__ __forceinline__ void cols_epilogue(int64_t u, int sub, int G, int W, float (&acc)[GV<T>::E], float ds,
                                              const float* __restrict__ dt, const float* __restrict__ asrc,
                                              const float* __restrict__ adst, T* __restrict__ dz,
                                              T* __restrict__ DS) {
    constexpr int E = GV<T>::E;
    const float dtu = dt[u];
    if (sub < G) {
#pragma unroll
        for (int q = 0; q < E; q++) {
            const int c = sub * E + q;
            acc[q] = fmaf(ds, asrc[c], fmaf(dtu, adst[c], acc[q]));
        }
        GV<T>::store(dz + u * W + sub * E, acc);
    }
    if (sub == 0) {
        float f[16];
#pragma unroll
        for (int q = 0; q < 16; q++) f[q] = 0.f;
        f[0] = ds; f[1] = dtu;
#pragma unroll
        for (int q = 0; q < 16; q += E) GV<T>::store(DS + u * 16 + q, f + q);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_gat_cols(int64_t n, const int4* __restrict__ desc, const int32_t* __restrict__ tcol,
                                                  const int32_t* __restrict__ eid, const T* __restrict__ z,
                                                  const T* __restrict__ g, const float* __restrict__ alpha,
                                                  const float* __restrict__ alpha_self, const float4* __restrict__ att,
                                                  const float* __restrict__ dt, const float* __restrict__ asrc,
                                                  const float* __restrict__ adst, T* __restrict__ dz, T* __restrict__ DS,
                                                  int W, int G, int G2) {
    constexpr int E = GV<T>::E;
    const int lane = threadIdx.x & 31;
    const int P = 32 / G2, slot = lane / G2, sub = lane % G2;
    const int64_t ri = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * P + slot;
    int64_t u = -1, e0 = 0, e1 = 0;
    if (ri < n) {
        const int4 d = __ldg(desc + ri);
        if (d.y <= kSegLen) {
            u = d.x;
            e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
            e1 = e0 + d.y;
        }
    }
    const int64_t len = e1 - e0;
    int64_t mx = len;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
    float zu[E], acc[E];
    float su = 0.f;
#pragma unroll
    for (int q = 0; q < E; q++) { zu[q] = 0.f; acc[q] = 0.f; }
    if (u >= 0) {
        if (sub < G) GV<T>::load(z + u * W + sub * E, zu);
        su = att[u].x;
    }
    float ds = 0.f;
    for (int64_t k = 0; k <= mx; k++) {
        // k < len: in-edge (v -> u); k == len: the self loop; beyond: idle
        const bool edge = k < len, self = k == len && u >= 0;
        const int64_t v = edge ? tcol[e0 + k] : (self ? u : 0);
        float gv[E];
        float p = 0.f;
        if ((edge || self) && sub < G) {
            GV<T>::load(g + v * W + sub * E, gv);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gv[q], zu[q], p);
        }
        const float dd = group_sum<T>(p, G2);
        if (edge || self) {
            const float a = edge ? alpha[eid[e0 + k]] : alpha_self[u];
            const float4 av = att[v];
            if (sub < G) {
#pragma unroll
                for (int q = 0; q < E; q++) acc[q] = fmaf(a, gv[q], acc[q]);
            }
            ds = fmaf(a * (dd - av.w), lrelu_d(su + av.y), ds);
        }
    }
    if (u >= 0) cols_epilogue<T>(u, sub, G, W, acc, ds, dt, asrc, adst, dz, DS);
}

template <typename T>
__global__ void __launch_bounds__(kHW * 32) k_gat_cols_heavy(const int32_t* __restrict__ heavy_rows,
                                                        const int64_t* __restrict__ trowptr, const int32_t* __restrict__ tcol,
                                                        const int32_t* __restrict__ eid, const T* __restrict__ z,
                                                        const T* __restrict__ g, const float* __restrict__ alpha,
                                                        const float* __restrict__ alpha_self, const float4* __restrict__ att,
                                                        const float* __restrict__ dt, const float* __restrict__ asrc,
                                                        const float* __restrict__ adst, T* __restrict__ dz, T* __restrict__ DS,
                                                        int W, int G, int G2) {
    constexpr int E = GV<T>::E;
    __shared__ float red[kHW][32 * 8 + 1];
    __shared__ float dsw[kHW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t u = heavy_rows[blockIdx.x];
    const int64_t r0 = trowptr[u], r1 = trowptr[u + 1], L = r1 - r0;
    const int P = 32 / G2, slot = lane / G2, sub = lane % G2;
    const int64_t w0 = r0 + L * w / kHW, w1 = r0 + L * (w + 1) / kHW;
    float zu[E], acc[E];
#pragma unroll
    for (int q = 0; q < E; q++) { zu[q] = 0.f; acc[q] = 0.f; }
    if (sub < G) GV<T>::load(z + u * W + sub * E, zu);
    const float su = att[u].x;
    float ds = 0.f;
    const int64_t trips = (w1 - w0 + P - 1) / P;
    for (int64_t k = 0; k < trips; k++) {
        const int64_t e = w0 + k * P + slot;
        const bool ok = e < w1;
        const int64_t v = ok ? tcol[e] : 0;
        float gv[E];
        float p = 0.f;
        if (ok && sub < G) {
            GV<T>::load(g + v * W + sub * E, gv);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gv[q], zu[q], p);
        }
        const float dd = group_sum<T>(p, G2);
        if (ok) {
            const float a = alpha[eid[e]];
            const float4 av = att[v];
            if (sub < G) {
#pragma unroll
                for (int q = 0; q < E; q++) acc[q] = fmaf(a, gv[q], acc[q]);
            }
            ds = fmaf(a * (dd - av.w), lrelu_d(su + av.y), ds);
        }
    }
    // combine the warp's groups (slot order), then the 8 warps (warp order)
    float t[E];
#pragma unroll
    for (int q = 0; q < E; q++) t[q] = 0.f;
    float tds = 0.f;
    for (int k = 0; k < P; k++) {
#pragma unroll
        for (int q = 0; q < E; q++) t[q] += __shfl_sync(0xffffffffu, acc[q], k * G2 + sub);
        tds += __shfl_sync(0xffffffffu, ds, k * G2);
    }
    if (slot == 0 && sub < G) {
#pragma unroll
        for (int q = 0; q < E; q++) red[w][sub * E + q] = t[q];
    }
    if (lane == 0) dsw[w] = tds;
    __syncthreads();
    if (w == 0 && slot == 0) {
        float s[E];
#pragma unroll
        for (int q = 0; q < E; q++) s[q] = 0.f;
        float sds = 0.f;
        for (int k = 0; k < kHW; k++) {
            if (sub < G) {
#pragma unroll
                for (int q = 0; q < E; q++) s[q] += red[k][sub * E + q];
            }
            sds += dsw[k];
        }
        // self loop
        float gu[E];
        float p = 0.f;
        if (sub < G) {
            GV<T>::load(g + u * W + sub * E, gu);
#pragma unroll
            for (int q = 0; q < E; q++) p = fmaf(gu[q], zu[q], p);
        }
        // group_sum over the G2 lanes of slot 0 (the other slots of warp 0 hold zeros)
        float dd = p;
        for (int o = G2 >> 1; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu >> (32 - G2) , dd, o);
        const float a = alpha_self[u];
        const float4 au = att[u];
        if (sub < G) {
#pragma unroll
            for (int q = 0; q < E; q++) s[q] = fmaf(a, gu[q], s[q]);
        }
        sds = fmaf(a * (dd - au.w), lrelu_d(su + au.y), sds);
        cols_epilogue<T>(u, sub, G, W, s, sds, dt, asrc, adst, dz, DS);
    }
}

// [da_src; da_dst] rows of the layer gradient from C = z^T [ds dt 0..] ([N x 16] fp32)
__global__ void k_gat_da(int K, int N, const float* __restrict__ C, float* __restrict__ dw) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        dw[(int64_t)K * N + j] = C[j * 16 + 0];
        dw[(int64_t)(K + 1) * N + j] = C[j * 16 + 1];
    }
}


// ------------------------------------------------------------------------------ host side
struct GatSaved { char* Z; float4* att; float *alpha, *alpha_self; size_t total; };
static inline size_t gal(size_t b) { return (b + 255) / 256 * 256; }
static GatSaved gat_saved_layout(const grappa_part* part, int f_out, grappa_dtype dt, void* base) {
    const size_t n = (size_t)part->info.n_core, nnz = (size_t)part->info.nnz, es = dt == GRAPPA_BF16 ? 2 : 4;
    char* b = (char*)base;
    GatSaved L{};
    size_t off = 0;
    L.Z = b + off; off += gal(n * f_out * es);
    L.att = (float4*)(b + off); off += gal(n * 16);
    L.alpha = (float*)(b + off); off += gal((nnz > 0 ? nnz : 1) * 4);
    L.alpha_self = (float*)(b + off); off += gal(n * 4);
    L.total = off;
    return L;
}
size_t gat_saved_bytes(const grappa_part* part, int f_out, grappa_dtype dt) {
    return gat_saved_layout(part, f_out, dt, nullptr).total;
}
struct GatWs { float* wext; float* partial; float* dtv; char* dZ; char* DS; float* C; float* splitk; int32_t* rev; size_t total; };
static GatWs gat_ws_layout(const grappa_part* part, int f_in, int f_out, grappa_dtype dt, void* base) {
    const size_t n = (size_t)part->info.n_core, es = dt == GRAPPA_BF16 ? 2 : 4;
    const size_t slots = (size_t)std::max<int64_t>(part->info.n_slots, part->t_n_slots);
    char* b = (char*)base;
    GatWs L{};
    size_t off = 0;
    L.wext = (float*)(b + off); off += gal((size_t)2 * f_in * 4);
    L.partial = (float*)(b + off); off += gal(slots * f_out * 4);
    L.dtv = (float*)(b + off); off += gal(n * 4);
    L.dZ = b + off; off += gal(n * f_out * es);
    L.DS = b + off; off += gal(n * 16 * es);
    L.C = (float*)(b + off); off += gal((size_t)f_out * 16 * 4);
    L.splitk = (float*)(b + off);
    off += gal(std::max(gemm_tn_ws_bytes(part->info.n_core, f_in, 0, f_out),
                        gemm_tn_ws_bytes(part->info.n_core, f_out, 0, 16)));
    L.total = off;
    return L;
}
size_t gat_ws_bytes(const grappa_part* part, int f_in, int f_out, grappa_dtype dt) {
    return gat_ws_layout(part, f_in, f_out, dt, nullptr).total;
}

static int pow2_ge(int x) { int p = 1; while (p < x) p <<= 1; return p; }

grappa_status gat_check(const grappa_part* part, int f_in, int f_out, grappa_dtype dt) {
    const int G = f_out * (dt == GRAPPA_BF16 ? 2 : 4) / 16;
    GRAPPA_ARG(G >= 1 && G <= 32, GRAPPA_E_SHAPE,
               "GAT: f_out = %d unsupported for this dtype (one 16-byte vector per lane, <= 32 lanes)", f_out);
    GRAPPA_ARG(part->info.nnz < (1ll << 31), GRAPPA_E_SHAPE, "GAT: nnz must fit int32 edge ids");
    (void)f_in;
    return GRAPPA_OK;
}

grappa_status gat_fwd(grappa_ctx* ctx, const grappa_part* part, int f_in, int f_out, int relu, const void* h_in,
                      const float* w, void* h_out, void* saved, void* ws, grappa_dtype dt, cudaStream_t s) {
    GRAPPA_TRY(gat_check(part, f_in, f_out, dt));
    const grappa_part_info& I = part->info;
    const int64_t n = I.n_core;
    GatSaved S = gat_saved_layout(part, f_out, dt, saved);
    GatWs Wk = gat_ws_layout(part, f_in, f_out, dt, ws);
    // wa = [W a_src; W a_dst];  att.{s, t} = h_in wa (fp32);  z = h_in W (kept in `saved`)
    k_gat_wa<<<(unsigned)ceil_div(2 * f_in, 128), 128, 0, s>>>(f_in, f_out, w, Wk.wext);
    GRAPPA_LAUNCHED(ctx);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), (int64_t)ctx->sm_count * 16));
    if (dt == GRAPPA_BF16)
        k_gat_st<__nv_bfloat16><<<grid, 256, 0, s>>>(n, f_in, (const __nv_bfloat16*)h_in, Wk.wext, S.att);
    else
        k_gat_st<float><<<grid, 256, 0, s>>>(n, f_in, (const float*)h_in, Wk.wext, S.att);
    GRAPPA_LAUNCHED(ctx);
    GemmArgs g;
    g.M = n; g.K1 = f_in; g.N = f_out; g.A1 = h_in; g.B = w; g.n_split = f_out; g.C1 = S.Z;
    GRAPPA_TRY(gemm_nn(ctx, g, dt, s));
    // attention coefficients
    k_gat_alpha<<<grid, 256, 0, s>>>(n, I.rowptr, I.col, S.alpha, S.alpha_self, S.att);
    GRAPPA_LAUNCHED(ctx);
    if (I.n_heavy > 0) {
        k_gat_alpha_heavy<<<(unsigned)I.n_heavy, kHW * 32, 0, s>>>((const int32_t*)part->heavy_rows.p, I.rowptr,
                                                                   I.col, S.alpha, S.alpha_self, S.att);
        GRAPPA_LAUNCHED(ctx);
    }
    // h_out = act(alpha_self z_v + sum alpha_e z_u): the SpMM with per-edge weights
    SpmmArgs a;
    a.X = S.Z; a.width = f_out; a.edge_w = S.alpha; a.self = 1; a.self_sep = 1; a.self_scale = S.alpha_self;
    a.relu = relu; a.out = h_out; a.partial = Wk.partial;
    return spmm(ctx, part, a, dt, s);
}

grappa_status gat_bwd(grappa_ctx* ctx, const grappa_part* part, int f_in, int f_out, int relu_in,
                      const void* dz_out, const void* h_in, const float* w, const void* saved, float* dw,
                      void* dz_in, void* ws, grappa_dtype dt, cudaStream_t s) {
    GRAPPA_TRY(gat_check(part, f_in, f_out, dt));
    const grappa_part_info& I = part->info;
    const int64_t n = I.n_core;
    GatSaved S = gat_saved_layout(part, f_out, dt, const_cast<void*>(saved));
    GatWs Wk = gat_ws_layout(part, f_in, f_out, dt, ws);
    grappa_part* mp = const_cast<grappa_part*>(part);
    // forward edge id of every transposed entry (cached in the part until the next repartition)
    if (!mp->t_eid_ready) {
        GRAPPA_TRY(mp->t_eid.grow((size_t)(I.nnz > 0 ? I.nnz : 1) * 4));
        k_gat_rev<<<(unsigned)ctx->sm_count * 16, 256, 0, s>>>(n, I.rowptr, I.col, (int32_t*)mp->t_eid.p);
        GRAPPA_LAUNCHED(ctx);
        mp->t_eid_ready = true;
    }
    const int32_t* eid = (const int32_t*)mp->t_eid.p;
    const int es = dt == GRAPPA_BF16 ? 2 : 4;
    const int G = f_out * es / 16, G2 = pow2_ge(G), P = 32 / G2;
    const unsigned grid = (unsigned)ceil_div(ceil_div(n, P), 8);
    const int64_t* trow = part->halo ? (const int64_t*)part->t_rowptr.p : I.rowptr;
    const int32_t* tcol = part->halo ? (const int32_t*)part->t_col.p : I.col;
    const int4* tdesc = (const int4*)(part->halo ? part->t_row_desc.p : part->row_desc.p);
    const int32_t* theavy = (const int32_t*)(part->halo ? part->t_heavy_rows.p : part->heavy_rows.p);
    const int64_t tn_heavy = part->halo ? part->t_n_heavy : I.n_heavy;
    const float* asrc = w + (int64_t)f_in * f_out;
    const float* adst = asrc + f_out;
    {
        ProfScope ps(ctx, s, GRAPPA_K_SPMM, (double)I.nnz * (4.0 + 4.0 + 16.0 + f_out * es) * 2.0,
                     4.0 * (double)I.nnz * f_out);
        if (dt == GRAPPA_BF16) {
            using T = __nv_bfloat16;
            if (n > 0) {
                k_gat_rows<T><<<grid, 256, 0, s>>>(n, (const int4*)part->row_desc.p, I.col, (const T*)S.Z,
                                                   (const T*)dz_out, S.alpha, S.alpha_self, S.att, Wk.dtv, f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (I.n_heavy > 0) {
                k_gat_rows_heavy<T><<<(unsigned)I.n_heavy, kHW * 32, 0, s>>>((const int32_t*)part->heavy_rows.p, I.rowptr,
                                                                        I.col, (const T*)S.Z, (const T*)dz_out, S.alpha,
                                                                        S.alpha_self, S.att, Wk.dtv, f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (n > 0) {
                k_gat_cols<T><<<grid, 256, 0, s>>>(n, tdesc, tcol, eid, (const T*)S.Z, (const T*)dz_out, S.alpha,
                                                   S.alpha_self, S.att, Wk.dtv, asrc, adst, (T*)Wk.dZ, (T*)Wk.DS,
                                                   f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (tn_heavy > 0) {
                k_gat_cols_heavy<T><<<(unsigned)tn_heavy, kHW * 32, 0, s>>>(theavy, trow, tcol, eid, (const T*)S.Z,
                                                                       (const T*)dz_out, S.alpha, S.alpha_self, S.att,
                                                                       Wk.dtv, asrc, adst, (T*)Wk.dZ, (T*)Wk.DS,
                                                                       f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
        } else {
            using T = float;
            if (n > 0) {
                k_gat_rows<T><<<grid, 256, 0, s>>>(n, (const int4*)part->row_desc.p, I.col, (const T*)S.Z,
                                                   (const T*)dz_out, S.alpha, S.alpha_self, S.att, Wk.dtv, f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (I.n_heavy > 0) {
                k_gat_rows_heavy<T><<<(unsigned)I.n_heavy, kHW * 32, 0, s>>>((const int32_t*)part->heavy_rows.p, I.rowptr,
                                                                        I.col, (const T*)S.Z, (const T*)dz_out, S.alpha,
                                                                        S.alpha_self, S.att, Wk.dtv, f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (n > 0) {
                k_gat_cols<T><<<grid, 256, 0, s>>>(n, tdesc, tcol, eid, (const T*)S.Z, (const T*)dz_out, S.alpha,
                                                   S.alpha_self, S.att, Wk.dtv, asrc, adst, (T*)Wk.dZ, (T*)Wk.DS,
                                                   f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
            if (tn_heavy > 0) {
                k_gat_cols_heavy<T><<<(unsigned)tn_heavy, kHW * 32, 0, s>>>(theavy, trow, tcol, eid, (const T*)S.Z,
                                                                       (const T*)dz_out, S.alpha, S.alpha_self, S.att,
                                                                       Wk.dtv, asrc, adst, (T*)Wk.dZ, (T*)Wk.DS,
                                                                       f_out, G, G2);
                GRAPPA_LAUNCHED(ctx);
            }
        }
    }
    // dW = h_in^T dz ; [da_src da_dst] = z^T [ds dt]
    GemmTNArgs t;
    t.M = n; t.K1 = f_in; t.N = f_out; t.A1 = h_in; t.B = Wk.dZ; t.C = dw; t.ws = Wk.splitk;
    GRAPPA_TRY(gemm_tn(ctx, t, dt, s));
    GemmTNArgs t2;
    t2.M = n; t2.K1 = f_out; t2.N = 16; t2.A1 = S.Z; t2.B = Wk.DS; t2.C = Wk.C; t2.ws = Wk.splitk;
    GRAPPA_TRY(gemm_tn(ctx, t2, dt, s));
    k_gat_da<<<1, 256, 0, s>>>(f_in, f_out, Wk.C, dw);
    GRAPPA_LAUNCHED(ctx);
    if (!dz_in) return GRAPPA_OK;
    // dh = dz W^T, gated by relu'(h_in)
    GemmArgs g;
    g.M = n; g.K1 = f_out; g.N = f_in; g.A1 = Wk.dZ; g.B = w; g.b_trans = 1;
    g.mask = relu_in ? h_in : nullptr; g.n_split = f_in; g.C1 = dz_in;
    return gemm_nn(ctx, g, dt, s);
}

}  // namespace grappa
