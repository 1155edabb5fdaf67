// spmm.cu -- partition-local neighbour aggregation (the SpMM of a4/a6).
//
// PAPER: P:141/P:177 (§3.2 isolated message passing over local nodes and edges only),
// P:435-437 (§5.1 GCN / GraphSAGE aggregation).
//
//   out[v] = epi( rs[v] * ( self * cs[v] * X[v] + sum_{u in N_loc(v)} cs[u] * X[u] ) )
//   epi(a) = relu?( (accumulate ? out_old[v] + a : a) * (mask ? 1[mask[v] > 0] : 1) )
//
//   GCN  fwd/bwd : rs = cs = (d_l+1)^-1/2, self = 1   (Dt^-1/2 (A+I) Dt^-1/2, symmetric)
//   SAGE fwd     : rs = 1/d_l, cs = 1, self = 0       (mean over local neighbours)
//   SAGE bwd     : rs = 1, cs = 1/d_l, self = 0, accumulate, mask = relu'(h_in)
//
// Design (B200): HBM-bound gather.  One warp per row; a row's W columns are covered by
// G = W/4 lanes holding 4 consecutive elements each (16 B fp32 / 8 B bf16 loads, fully
// coalesced per gathered row); the warp's 32/G lane groups ("slots") take different
// neighbours, and UNROLL neighbours per slot are in flight at once.  Column indices and the
// per-neighbour scale are loaded 32 at a time by the warp and broadcast with shuffles.
// Rows with d_l > kSegLen are split into kSegLen-edge segments (one warp each) whose fp32
// partial sums are combined in segment order by k_spmm_fixup: power-law hubs do not
// serialise a warp, and the result stays deterministic (no atomics).
#include "part.cuh"
#include "spmm.cuh"

namespace grappa {

template <typename T> struct Vec4;
template <> struct Vec4<float> {
    using type = float4;
    __device__ static float4 load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ static void to_f(const float4& v, float* f) { f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w; }
    __device__ static float4 from_f(const float* f) { return make_float4(f[0], f[1], f[2], f[3]); }
    __device__ static void store(float* p, const float* f) { *reinterpret_cast<float4*>(p) = from_f(f); }
};
template <> struct Vec4<__nv_bfloat16> {
    using type = uint2;
    __device__ static uint2 load(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
    __device__ static void to_f(const uint2& v, float* f) {
        __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
        float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
        f[0] = fa.x; f[1] = fa.y; f[2] = fb.x; f[3] = fb.y;
    }
    __device__ static void store(__nv_bfloat16* p, const float* f) {
        __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]);
        __nv_bfloat162 b = __floats2bfloat162_rn(f[2], f[3]);
        uint2 v;
        v.x = *reinterpret_cast<uint32_t*>(&a);
        v.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(p) = v;
    }
};

constexpr int kUnroll = 4;

// Gather-sum of edges [e0, e1) of one row into acc (lanes of slot `slot`, sub-lane `sub`).
template <typename T, int CPL>
__device__ __forceinline__ void gather_edges(const SpmmArgs& a, int64_t e0, int64_t e1, int lane,
                                             int G, int P, int slot, int sub, int W4,
                                             float (&acc)[CPL][4]) {
    const T* X = reinterpret_cast<const T*>(a.X);
    for (int64_t base = e0; base < e1; base += 32) {
        const int cnt = (int)((e1 - base) < 32 ? (e1 - base) : 32);
        int my_idx = 0;
        float my_w = 1.f;
        if (lane < cnt) {
            my_idx = a.col[base + lane];
            if (a.col_scale) my_w = a.col_scale[my_idx];
        }
        for (int j = 0; j < cnt; j += P * kUnroll) {
            typename Vec4<T>::type v[kUnroll][CPL];
            float wt[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                const int jj = j + u * P + slot;
                const int src = __shfl_sync(0xffffffffu, my_idx, jj & 31);
                const float w = __shfl_sync(0xffffffffu, my_w, jj & 31);
                const bool ok = (slot < P) && (jj < cnt);
                wt[u] = ok ? w : 0.f;
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    const int col4 = sub + c * G;
                    if (ok && col4 < W4)
                        v[u][c] = Vec4<T>::load(X + ((int64_t)src * W4 + col4) * 4);
                    else
                        v[u][c] = {};
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; u++)
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    float f[4];
                    Vec4<T>::to_f(v[u][c], f);
#pragma unroll
                    for (int q = 0; q < 4; q++) acc[c][q] = fmaf(wt[u], f[q], acc[c][q]);
                }
        }
    }
}

// Combine the P slot accumulators into slot 0 (lanes 0..G-1), in slot order.
template <int CPL>
__device__ __forceinline__ void reduce_slots(float (&acc)[CPL][4], int G, int P) {
    float tot[CPL][4];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < 4; q++) tot[c][q] = acc[c][q];
    for (int k = 1; k < P; k++) {
#pragma unroll
        for (int c = 0; c < CPL; c++)
#pragma unroll
            for (int q = 0; q < 4; q++) tot[c][q] += __shfl_down_sync(0xffffffffu, acc[c][q], k * G);
    }
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[c][q] = tot[c][q];
}

template <typename T, int CPL>
__device__ __forceinline__ void epilogue(const SpmmArgs& a, int64_t v, int sub, int G, int W4,
                                         float (&acc)[CPL][4]) {
    const T* X = reinterpret_cast<const T*>(a.X);
    T* out = reinterpret_cast<T*>(a.out);
    const T* mask = reinterpret_cast<const T*>(a.mask);
    const float rs = a.row_scale ? a.row_scale[v] : 1.f;
    const float cs = a.col_scale ? a.col_scale[v] : 1.f;
#pragma unroll
    for (int c = 0; c < CPL; c++) {
        const int col4 = sub + c * G;
        if (col4 >= W4) continue;
        const int64_t off = ((int64_t)v * W4 + col4) * 4;
        float r[4];
#pragma unroll
        for (int q = 0; q < 4; q++) r[q] = acc[c][q];
        if (a.self) {
            float f[4];
            Vec4<T>::to_f(Vec4<T>::load(X + off), f);
#pragma unroll
            for (int q = 0; q < 4; q++) r[q] = fmaf(cs, f[q], r[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) r[q] *= rs;
        if (a.accumulate) {
            float f[4];
            Vec4<T>::to_f(*reinterpret_cast<const typename Vec4<T>::type*>(out + off), f);
#pragma unroll
            for (int q = 0; q < 4; q++) r[q] += f[q];
        }
        if (mask) {
            float f[4];
            Vec4<T>::to_f(Vec4<T>::load(mask + off), f);
#pragma unroll
            for (int q = 0; q < 4; q++) r[q] = f[q] > 0.f ? r[q] : 0.f;
        }
        if (a.relu) {
#pragma unroll
            for (int q = 0; q < 4; q++) r[q] = fmaxf(r[q], 0.f);
        }
        Vec4<T>::store(out + off, r);
    }
}

template <typename T, int CPL>
__global__ void __launch_bounds__(256) k_spmm(SpmmArgs a, int G, int P) {
    const int lane = threadIdx.x & 31;
    const int64_t vrow = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int W4 = a.width / 4;
    const int slot = lane / G, sub = lane % G;
    float acc[CPL][4];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[c][q] = 0.f;
    if (vrow < a.n_slots) {
        // one kSegLen segment of a split row -> fp32 partial, combined by k_spmm_fixup
        const int32_t r = a.slot_row[vrow], sg = a.slot_seg[vrow];
        const int64_t e0 = a.rowptr[r] + (int64_t)sg * kSegLen;
        const int64_t e1 = min(a.rowptr[r + 1], e0 + kSegLen);
        gather_edges<T, CPL>(a, e0, e1, lane, G, P, slot, sub, W4, acc);
        reduce_slots<CPL>(acc, G, P);
        if (lane < G) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int col4 = sub + c * G;
                if (col4 < W4)
                    *reinterpret_cast<float4*>(a.partial + (vrow * W4 + col4) * 4) =
                        make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
            }
        }
        return;
    }
    const int64_t v = vrow - a.n_slots;
    if (v >= a.n) return;
    const int64_t e0 = a.rowptr[v], e1 = a.rowptr[v + 1];
    if (e1 - e0 > kSegLen) return;              // split row: finished by the fix-up kernel
    gather_edges<T, CPL>(a, e0, e1, lane, G, P, slot, sub, W4, acc);
    reduce_slots<CPL>(acc, G, P);
    if (lane < G) epilogue<T, CPL>(a, v, sub, G, W4, acc);
}

template <typename T, int CPL>
__global__ void __launch_bounds__(256) k_spmm_fixup(SpmmArgs a, int G) {
    const int lane = threadIdx.x & 31;
    const int64_t h = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (h >= a.n_heavy) return;
    const int W4 = a.width / 4;
    const int32_t r = a.heavy_rows[h];
    const int s0 = a.heavy_slot_off[h], s1 = a.heavy_slot_off[h + 1];
    float acc[CPL][4];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[c][q] = 0.f;
    if (lane >= G) return;
    for (int sl = s0; sl < s1; sl++) {
#pragma unroll
        for (int c = 0; c < CPL; c++) {
            const int col4 = lane + c * G;
            if (col4 < W4) {
                float4 p = *reinterpret_cast<const float4*>(a.partial + ((int64_t)sl * W4 + col4) * 4);
                acc[c][0] += p.x; acc[c][1] += p.y; acc[c][2] += p.z; acc[c][3] += p.w;
            }
        }
    }
    epilogue<T, CPL>(a, r, lane, G, W4, acc);
}

template <typename T, int CPL>
static grappa_status launch_cpl(grappa_ctx* ctx, const SpmmArgs& a, int G, int P, cudaStream_t s) {
    const int64_t vrows = a.n + a.n_slots;
    if (vrows > 0) {
        k_spmm<T, CPL><<<(unsigned)ceil_div(vrows, 8), 256, 0, s>>>(a, G, P);
        GRAPPA_LAUNCHED(ctx);
    }
    if (a.n_heavy > 0) {
        k_spmm_fixup<T, CPL><<<(unsigned)ceil_div(a.n_heavy, 8), 256, 0, s>>>(a, G);
        GRAPPA_LAUNCHED(ctx);
    }
    return GRAPPA_OK;
}

template <typename T>
static grappa_status launch_t(grappa_ctx* ctx, const SpmmArgs& a, cudaStream_t s) {
    const int W4 = a.width / 4;
    const int G = W4 <= 32 ? W4 : 32;
    const int P = 32 / G;
    const int cpl = (W4 + G - 1) / G;
    if (cpl <= 1) return launch_cpl<T, 1>(ctx, a, G, P, s);
    if (cpl <= 2) return launch_cpl<T, 2>(ctx, a, G, P, s);
    if (cpl <= 4) return launch_cpl<T, 4>(ctx, a, G, P, s);
    if (cpl <= 8) return launch_cpl<T, 8>(ctx, a, G, P, s);
    if (cpl <= 12) return launch_cpl<T, 12>(ctx, a, G, P, s);
    set_error("spmm: width %d too large", a.width);
    return GRAPPA_E_SHAPE;
}

grappa_status spmm(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                   cudaStream_t s) {
    const grappa_part_info& I = part->info;
    a.n = I.n_core;
    a.rowptr = I.rowptr;
    a.col = I.col;
    a.n_slots = I.n_slots;
    a.n_heavy = I.n_heavy;
    a.slot_row = (const int32_t*)part->slot_row.p;
    a.slot_seg = (const int32_t*)part->slot_seg.p;
    a.heavy_rows = (const int32_t*)part->heavy_rows.p;
    a.heavy_slot_off = (const int32_t*)part->heavy_slot_off.p;
    if (a.width % 4 != 0) {
        set_error("spmm: width %d not a multiple of 4", a.width);
        return GRAPPA_E_SHAPE;
    }
    const double es = dt == GRAPPA_BF16 ? 2.0 : 4.0, w = a.width, nnz = (double)I.nnz;
    const double per_edge = 4.0 + (a.col_scale ? 4.0 : 0.0) + w * es;
    const double per_row = 8.0 + (a.row_scale ? 4.0 : 0.0) + (a.col_scale ? 4.0 : 0.0) +
                           (a.self ? w * es : 0.0) + w * es + (a.accumulate ? w * es : 0.0) +
                           (a.mask ? w * es : 0.0);
    ProfScope ps(ctx, s, GRAPPA_K_SPMM, nnz * per_edge + (double)I.n_core * per_row, 2.0 * nnz * w);
    return dt == GRAPPA_BF16 ? launch_t<__nv_bfloat16>(ctx, a, s) : launch_t<float>(ctx, a, s);
}

}  // namespace grappa
