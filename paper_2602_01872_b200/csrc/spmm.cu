// spmm.cu -- partition-local neighbour aggregation (the SpMM of a4/a6).
//
// PAPER: P:141/P:177 (§3.2 isolated message passing over local nodes and edges only),
// P:435-437 (§5.1 GCN / GraphSAGE aggregation).
//
//   out[v] = epi( rs[v] * ( self * ss[v] * X[v] + ns[v] * sum_{u in N_loc(v)} cs[u] * X[u] ) )
//   ss = cs unless self_sep (then self_scale, or 1); ns = nbr_scale or 1 (node-level, R30)
//   epi(a) = relu?( (accumulate ? out_old[v] + a : a) * (mask ? 1[mask[v] > 0] : 1) )
//
//   GCN  fwd/bwd : rs = cs = (d_l+1)^-1/2, self = 1   (Dt^-1/2 (A+I) Dt^-1/2, symmetric)
//   SAGE fwd     : rs = 1/d_l, cs = 1, self = 0       (mean over local neighbours)
//   SAGE bwd     : rs = 1, cs = 1/d_l, self = 0, accumulate, mask = relu'(h_in)
//
// Design (B200): HBM-bound gather.  One warp per row; a row's W elements are covered by
// G = W/EPV lanes each holding one 16-byte vector (EPV = 4 fp32 or 8 bf16), so every gathered
// neighbour row is one fully coalesced 16 B x G transaction; the warp's 32/G lane groups
// ("slots") take different neighbours and kUnroll neighbours per slot are in flight at once.
// Column indices and per-neighbour scales are loaded 32 at a time by the warp and broadcast
// with shuffles.  Rows with d_l > kSegLen are split into kSegLen-edge segments (one warp
// each) whose fp32 partial sums are combined in segment order by k_spmm_fixup: power-law
// hubs do not serialise a warp and the result stays bitwise deterministic (no atomics).
#include "part.cuh"
#include "spmm.cuh"
#include "tc.cuh"

namespace grappa {

template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int EPV = 4;
    using type = float4;
    __device__ static float4 load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ static float4 load_ordered(const float* p) { return load(p); }
    __device__ static float4 load_rw(const float* p) { return *reinterpret_cast<const float4*>(p); }
    __device__ static void to_f(const float4& v, float* f) { f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w; }
    __device__ static void store(float* p, const float* f) {
        *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int EPV = 8;
    using type = uint4;
    __device__ static uint4 load(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
    // same load as an ordered (volatile) instruction, see acc_bf16
    __device__ static uint4 load_ordered(const __nv_bfloat16* p) {
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        return v;
    }
    __device__ static uint4 load_rw(const __nv_bfloat16* p) { return *reinterpret_cast<const uint4*>(p); }
    __device__ static void to_f(const uint4& v, float* f) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            // bf16 -> fp32 is a 16-bit shift
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
};

constexpr int kUnroll = 4;


// (a0, a1) += w * (x0, x1) as one packed FFMA2 (sm_100): halves the FMA issue count of the
// gather-accumulate loop, whose instruction issue -- not DRAM -- is the limiter (ncu)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w, float x0, float x1) {
    asm("{\n\t.reg .b64 a, x, ww;\n\t"
        "mov.b64 a, {%0, %1};\n\t"
        "mov.b64 x, {%2, %3};\n\t"
        "mov.b64 ww, {%4, %4};\n\t"
        "fma.rn.f32x2 a, x, ww, a;\n\t"
        "mov.b64 {%0, %1}, a;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(x0), "f"(x1), "f"(w));
}
// dispatch knob (tests / A-B timing) for narrow rows: 0 = row-group kernel with 4 feature
// loads in flight per lane (default; measured best), 1 = warp-per-row kernel, 2 = row-group
// kernel with 8 loads in flight (more registers, fewer resident warps: slower on B200),
// 3 = row-group kernel over the rows in natural order (no degree bucketing)
static int g_spmm_variant = 0;
void spmm_force_warp_per_row(int v) { g_spmm_variant = v; }
// unweighted bf16 rows: 32-byte lanes (1) or the 16-byte row-group kernel (0, default: measured
// faster on products -- the 32-byte kernel needs ~2x the registers, halving resident warps)
static int g_wide_loads = 0;
void spmm_set_wide(int v) { g_wide_loads = v; }

// Gather-sum of edges [e0, e1) of one row into acc (lanes of slot `slot`, sub-lane `sub`).
template <typename T, int CPL>
__device__ __forceinline__ void gather_edges(const SpmmArgs& a, int64_t e0, int64_t e1, int lane,
                                             int G, int P, int slot, int sub, int WV,
                                             float (&acc)[CPL][Vec<T>::EPV]) {
    constexpr int E = Vec<T>::EPV;
    const T* X = reinterpret_cast<const T*>(a.X);
    for (int64_t base = e0; base < e1; base += 32) {
        const int cnt = (int)((e1 - base) < 32 ? (e1 - base) : 32);
        int my_idx = 0;
        float my_w = 1.f;
        if (lane < cnt) {
            my_idx = a.col[base + lane];
            if (a.edge_w) my_w = a.edge_w[base + lane];
            else if (a.col_scale) my_w = a.col_scale[my_idx];
        }
        for (int j = 0; j < cnt; j += P * kUnroll) {
            typename Vec<T>::type v[kUnroll][CPL];
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
                    const int cv = sub + c * G;
                    if (ok && cv < WV)
                        v[u][c] = Vec<T>::load(X + ((int64_t)src * WV + cv) * E);
                    else
                        v[u][c] = {};
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; u++)
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    float f[E];
                    Vec<T>::to_f(v[u][c], f);
#pragma unroll
                    for (int q = 0; q < E; q++) acc[c][q] = fmaf(wt[u], f[q], acc[c][q]);
                }
        }
    }
}

// Combine the P slot accumulators into slot 0 (lanes 0..G-1), in slot order.
template <int CPL, int E>
__device__ __forceinline__ void reduce_slots(float (&acc)[CPL][E], int G, int P) {
    float tot[CPL][E];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < E; q++) tot[c][q] = acc[c][q];
    for (int k = 1; k < P; k++) {
#pragma unroll
        for (int c = 0; c < CPL; c++)
#pragma unroll
            for (int q = 0; q < E; q++) tot[c][q] += __shfl_down_sync(0xffffffffu, acc[c][q], k * G);
    }
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < E; q++) acc[c][q] = tot[c][q];
}

template <typename T, int CPL>
__device__ __forceinline__ void epilogue(const SpmmArgs& a, int64_t v, int64_t ov, int sub, int G,
                                         int WV, float (&acc)[CPL][Vec<T>::EPV]) {
    constexpr int E = Vec<T>::EPV;
    const T* X = reinterpret_cast<const T*>(a.X);
    T* out = reinterpret_cast<T*>(a.out);
    const T* mask = reinterpret_cast<const T*>(a.mask);
    const float rs = a.row_scale ? a.row_scale[v] : 1.f;
    // self coefficient: read only when there is a self term (on a rectangular block, e.g. the
    // mini-batch transpose, col_scale is indexed by the other side and v may be out of its range)
    const float cs = !a.self ? 0.f
                     : a.self_sep ? (a.self_scale ? a.self_scale[v] : 1.f) : (a.col_scale ? a.col_scale[v] : 1.f);
    const float ns = a.nbr_scale ? a.nbr_scale[v] : 1.f;
#pragma unroll
    for (int c = 0; c < CPL; c++) {
        const int cv = sub + c * G;
        if (cv >= WV) continue;
        const int64_t off = ((int64_t)v * WV + cv) * E;
        const int64_t ooff = ((int64_t)ov * WV + cv) * E;
        float r[E];
#pragma unroll
        for (int q = 0; q < E; q++) r[q] = acc[c][q];
        if (a.nbr_scale) {
#pragma unroll
            for (int q = 0; q < E; q++) r[q] *= ns;
        }
        if (a.self) {
            float f[E];
            Vec<T>::to_f(Vec<T>::load(X + off), f);
#pragma unroll
            for (int q = 0; q < E; q++) r[q] = fmaf(cs, f[q], r[q]);
        }
#pragma unroll
        for (int q = 0; q < E; q++) r[q] *= rs;
        if (a.accumulate) {
            float f[E];
            Vec<T>::to_f(Vec<T>::load_rw(out + ooff), f);
#pragma unroll
            for (int q = 0; q < E; q++) r[q] += f[q];
        }
        if (mask) {
            float f[E];
            Vec<T>::to_f(Vec<T>::load(mask + off), f);
#pragma unroll
            for (int q = 0; q < E; q++) r[q] = f[q] > 0.f ? r[q] : 0.f;
        }
        if (a.relu) {
#pragma unroll
            for (int q = 0; q < E; q++) r[q] = fmaxf(r[q], 0.f);
        }
        Vec<T>::store(out + ooff, r);
    }
}

template <typename T, int CPL>
__global__ void __launch_bounds__(256) k_spmm(SpmmArgs a, int G, int P) {
    constexpr int E = Vec<T>::EPV;
    const int lane = threadIdx.x & 31;
    const int64_t vrow = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int WV = a.width / E;
    const int slot = lane / G, sub = lane % G;
    float acc[CPL][E];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < E; q++) acc[c][q] = 0.f;
    if (vrow < a.n_slots) {
        // one kSegLen segment of a split row -> fp32 partial, combined by k_spmm_fixup
        const int32_t r = a.slot_row[vrow], sg = a.slot_seg[vrow];
        const int64_t e0 = a.rowptr[r] + (int64_t)sg * kSegLen;
        const int64_t e1 = min(a.rowptr[r + 1], e0 + kSegLen);
        gather_edges<T, CPL>(a, e0, e1, lane, G, P, slot, sub, WV, acc);
        reduce_slots<CPL, E>(acc, G, P);
        if (lane < G) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int cv = sub + c * G;
                if (cv < WV) {
                    float* dst = a.partial + ((int64_t)vrow * WV + cv) * E;
#pragma unroll
                    for (int q = 0; q < E; q += 4)
                        *reinterpret_cast<float4*>(dst + q) =
                            make_float4(acc[c][q], acc[c][q + 1], acc[c][q + 2], acc[c][q + 3]);
                }
            }
        }
        return;
    }
    const int64_t v = vrow - a.n_slots;
    if (v >= a.n) return;
    const int64_t e0 = a.rowptr[v], e1 = a.rowptr[v + 1];
    if (e1 - e0 > kSegLen) return;              // split row: finished by the fix-up kernel
    gather_edges<T, CPL>(a, e0, e1, lane, G, P, slot, sub, WV, acc);
    reduce_slots<CPL, E>(acc, G, P);
    if (lane < G) epilogue<T, CPL>(a, v, v, sub, G, WV, acc);
}

template <typename T, int CPL>
__global__ void __launch_bounds__(256) k_spmm_fixup(SpmmArgs a, int G) {
    constexpr int E = Vec<T>::EPV;
    const int lane = threadIdx.x & 31;
    const int64_t h = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (h >= a.n_heavy) return;
    const int WV = a.width / E;
    const int32_t r = a.heavy_rows[h];
    const int s0 = a.heavy_slot_off[h], s1 = a.heavy_slot_off[h + 1];
    float acc[CPL][E];
#pragma unroll
    for (int c = 0; c < CPL; c++)
#pragma unroll
        for (int q = 0; q < E; q++) acc[c][q] = 0.f;
    if (lane >= G) return;
    for (int sl = s0; sl < s1; sl++) {
#pragma unroll
        for (int c = 0; c < CPL; c++) {
            const int cv = lane + c * G;
            if (cv < WV) {
                const float* src = a.partial + ((int64_t)sl * WV + cv) * E;
#pragma unroll
                for (int q = 0; q < E; q += 4) {
                    const float4 p = *reinterpret_cast<const float4*>(src + q);
                    acc[c][q] += p.x; acc[c][q + 1] += p.y; acc[c][q + 2] += p.z; acc[c][q + 3] += p.w;
                }
            }
        }
    }
    epilogue<T, CPL>(a, r, a.out_compact ? h : r, lane, G, WV, acc);
}

// acc[0..7] += the 8 bf16 of v, each added to its fp32 accumulator by one mixed-precision
// FADD (add.rn.f32.bf16 -> FHADD.BF16, sm_100): no unpack instructions, no edge weight
__device__ __forceinline__ void acc_bf16(float (&acc)[8], const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
        unsigned short lo, hi;
        asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w[i]));
        // volatile: keeps the adds behind all U loads of the batch (the compiler would
        // otherwise hoist each add next to its load and serialise the gathers)
        asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc[2 * i]) : "h"(lo));
        asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc[2 * i + 1]) : "h"(hi));
    }
}
__device__ __forceinline__ void acc_plain(float (&acc)[8], const uint4& v) { acc_bf16(acc, v); }
__device__ __forceinline__ void acc_plain(float (&acc)[4], const float4& v) {
    acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
}

// Gather-accumulate of one row per lane group (narrow rows, W/EPV <= 32 vectors): every
// group of G lanes owns a row, lane `sub` holds one 16-byte vector of it.  Each lane
// prefetches R column indices (chunk = G*R edges) and U feature vectors are in flight per
// lane.  All 32 lanes must call it (shuffles); lanes with deg = 0 just follow along.
template <typename T, int R, int U, bool WT>
__device__ __forceinline__ void grp_accumulate(const T* __restrict__ X, const int32_t* __restrict__ col,
                                               const float* __restrict__ col_scale, int64_t e0,
                                               int deg, int G, int slot, int sub,
                                               float (&acc)[Vec<T>::EPV],
                                               const float* __restrict__ edge_w = nullptr) {
    constexpr int E = Vec<T>::EPV;
    const int WV = G;
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    const int CH = G * R;
    for (int off = 0; off < maxdeg; off += CH) {
        int idx[R];
        float wt[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int p = off + r * G + sub;
            const bool ok = p < deg;
            idx[r] = ok ? col[e0 + p] : 0;
            if (WT) wt[r] = ok ? (edge_w ? edge_w[e0 + p] : col_scale[idx[r]]) : 0.f;
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int jmax = min(G, maxdeg - off - r * G);
            for (int j = 0; j < jmax; j += U) {
                typename Vec<T>::type v[U];
                float w[U];
                // issue all U feature-row loads first (they need only the index), then fetch
                // the edge weights, so the weight gather's latency hides under the loads
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int jj = j + u;
                    const int srcl = slot * G + (jj < G ? jj : 0);
                    const int s = __shfl_sync(0xffffffffu, idx[r], srcl);
                    const bool ok = jj < G && off + r * G + jj < deg;
                    if (ok) v[u] = WT ? Vec<T>::load(X + ((int64_t)s * WV + sub) * E)
                                      : Vec<T>::load_ordered(X + ((int64_t)s * WV + sub) * E);
                    else v[u] = {};
                }
                if (WT) {
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int jj = j + u;
                        const int srcl = slot * G + (jj < G ? jj : 0);
                        const float ww = __shfl_sync(0xffffffffu, wt[r], srcl);
                        w[u] = (jj < G && off + r * G + jj < deg) ? ww : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        float f[E];
                        Vec<T>::to_f(v[u], f);
#pragma unroll
                        for (int q = 0; q < E; q += 2) ffma2(acc[q], acc[q + 1], w[u], f[q], f[q + 1]);
                    }
                } else {
                    // masked-off slots loaded zeros (v[u] = {}), so a plain add is exact
#pragma unroll
                    for (int u = 0; u < U; u++) acc_plain(acc, v[u]);
                }
            }
        }
    }
}

// Narrow rows: every group of G = W/EPV lanes owns a different row, so a warp carries
// P = 32/G independent rows and their dependent load chains (rowptr -> col -> scale /
// feature row) overlap; no cross-group reduction is needed.
template <typename T, int R, int U, bool WT>
__global__ void __launch_bounds__(256) k_spmm_grp(SpmmArgs a, int G, int P) {
    constexpr int E = Vec<T>::EPV;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int slot = lane / G, sub = lane - slot * G;
    const int WV = G;
    const int64_t vrow = warp * P + slot;
    int64_t e0 = 0, e1 = 0, orow = -1;
    bool to_partial = false;
    if (slot < P) {
        if (vrow < a.n_slots) {
            const int32_t r = a.slot_row[vrow], sg = a.slot_seg[vrow];
            e0 = a.rowptr[r] + (int64_t)sg * kSegLen;
            e1 = min(a.rowptr[r + 1], e0 + kSegLen);
            orow = vrow;
            to_partial = true;
        } else if (vrow - a.n_slots < a.n) {
            int64_t v;
            if (a.row_desc) {
                const int4 d = __ldg(a.row_desc + (vrow - a.n_slots));
                v = d.x;
                e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
                e1 = e0 + d.y;
            } else {
                v = a.row_order ? (int64_t)a.row_order[vrow - a.n_slots] : vrow - a.n_slots;
                e0 = a.rowptr[v];
                e1 = a.rowptr[v + 1];
            }
            if (e1 - e0 > kSegLen) e1 = e0;          // split row: finished by the fix-up kernel
            else orow = v;
        }
    }
    float acc[E];
#pragma unroll
    for (int q = 0; q < E; q++) acc[q] = 0.f;
    grp_accumulate<T, R, U, WT>(reinterpret_cast<const T*>(a.X), a.col, a.col_scale, e0, (int)(e1 - e0),
                                G, slot, sub, acc, a.edge_w);
    if (orow < 0) return;
    if (to_partial) {
        float* dst = a.partial + ((int64_t)orow * WV + sub) * E;
#pragma unroll
        for (int q = 0; q < E; q += 4)
            *reinterpret_cast<float4*>(dst + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
        return;
    }
    float acc1[1][E];
#pragma unroll
    for (int q = 0; q < E; q++) acc1[0][q] = acc[q];
    epilogue<T, 1>(a, orow, orow, sub, G, WV, acc1);
}

// 32-byte variant for unweighted bf16 rows (pre-scaled inputs): each lane owns 16 consecutive
// features and fetches them with one 256-bit load (LDG.E.ENL2.256), so a gathered row costs
// half the load, shuffle and address instructions of the 16-byte layout; G = width/16 lanes
// per row, P = 32/G rows per warp.
__device__ __forceinline__ void ld256(const __nv_bfloat16* p, uint4& a, uint4& b) {
    asm volatile("ld.global.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}

template <int R, int U>
__device__ __forceinline__ void grp_accumulate16(const __nv_bfloat16* __restrict__ X, const int32_t* __restrict__ col,
                                                 int64_t e0, int deg, int G, int slot, int P, int sub,
                                                 float (&lo)[8], float (&hi)[8]) {
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    // lanes of idle slots do not constrain the fast path
    const int mindeg = __reduce_min_sync(0xffffffffu, slot < P ? deg : 0x7fffffff);
    const int CH = G * R;
    const __nv_bfloat16* Xs = X + sub * 16;
    const int64_t rowel = (int64_t)G * 16;                 // elements per row
    for (int off = 0; off < maxdeg; off += CH) {
        int idx[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int p = off + r * G + sub;
            idx[r] = p < deg ? col[e0 + p] : 0;
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int base = off + r * G;
            const int jmax = min(G, maxdeg - base);        // batches any lane needs
            const int jfull = min(G, mindeg - base);       // batches every lane needs
            const int lim = deg - base;                    // this lane's valid edges
            for (int j = 0; j < jmax; j += U) {
                uint4 va[U], vb[U];
                if (j + U <= jfull) {
                    // full batch for the whole warp: no predication
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int s = __shfl_sync(0xffffffffu, idx[r], slot * G + j + u);
                        ld256(Xs + (int64_t)s * rowel, va[u], vb[u]);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int jj = j + u;
                        const int s = __shfl_sync(0xffffffffu, idx[r], (slot * G + jj) & 31);
                        if (jj < G && jj < lim) ld256(Xs + (int64_t)s * rowel, va[u], vb[u]);
                        else va[u] = vb[u] = make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    acc_bf16(lo, va[u]);
                    acc_bf16(hi, vb[u]);
                }
            }
        }
    }
}

template <int R, int U>
__global__ void __launch_bounds__(256) k_spmm_grp16(SpmmArgs a, int G, int P) {
    using T = __nv_bfloat16;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int slot = lane / G, sub = lane - slot * G;
    const int WV = 2 * G;                              // 8-element vectors per row
    const int64_t vrow = warp * P + slot;
    int64_t e0 = 0, e1 = 0, orow = -1;
    bool to_partial = false;
    if (slot < P) {
        if (vrow < a.n_slots) {
            const int32_t r = a.slot_row[vrow], sg = a.slot_seg[vrow];
            e0 = a.rowptr[r] + (int64_t)sg * kSegLen;
            e1 = min(a.rowptr[r + 1], e0 + kSegLen);
            orow = vrow;
            to_partial = true;
        } else if (vrow - a.n_slots < a.n) {
            const int64_t v = a.row_order ? (int64_t)a.row_order[vrow - a.n_slots] : vrow - a.n_slots;
            e0 = a.rowptr[v];
            e1 = a.rowptr[v + 1];
            if (e1 - e0 > kSegLen) e1 = e0;          // split row: finished by the fix-up kernel
            else orow = v;
        }
    }
    float lo[8], hi[8];
#pragma unroll
    for (int q = 0; q < 8; q++) lo[q] = hi[q] = 0.f;
    grp_accumulate16<R, U>(reinterpret_cast<const T*>(a.X), a.col, e0, (int)(e1 - e0), G, slot, P, sub, lo, hi);
    if (orow < 0) return;
    if (to_partial) {
        float* dst = a.partial + ((int64_t)orow * WV + 2 * sub) * 8;
#pragma unroll
        for (int q = 0; q < 8; q += 4) {
            *reinterpret_cast<float4*>(dst + q) = make_float4(lo[q], lo[q + 1], lo[q + 2], lo[q + 3]);
            *reinterpret_cast<float4*>(dst + 8 + q) = make_float4(hi[q], hi[q + 1], hi[q + 2], hi[q + 3]);
        }
        return;
    }
    float l1[1][8], h1[1][8];
#pragma unroll
    for (int q = 0; q < 8; q++) { l1[0][q] = lo[q]; h1[0][q] = hi[q]; }
    epilogue<T, 1>(a, orow, orow, 2 * sub, G, WV, l1);
    epilogue<T, 1>(a, orow, orow, 2 * sub + 1, G, WV, h1);
}

// split-row combine, one launch per SpMM call, one block per split row.  Rows of <= kFixWarps
// segments (almost all: 2-3 segments): warp 0 sums the slots in order; longer rows (hubs): warp
// w sums slots s0+w, s0+w+kFixWarps, ... in order, then the warp sums are added in warp order.
// For <= kFixWarps segments both orders are the same sum.  (A separate warp-per-row launch for
// the short rows cost one more kernel boundary per SpMM call.)
constexpr int kFixWarps = 8;
template <typename T>
__global__ void __launch_bounds__(kFixWarps * 32) k_spmm_fixup_blk(SpmmArgs a, int G) {
    constexpr int E = Vec<T>::EPV;
    __shared__ float red[kFixWarps][32 * E];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t h = blockIdx.x;
    const int WV = G;
    const int32_t r = a.heavy_rows[h];
    const int s0 = a.heavy_slot_off[h], s1 = a.heavy_slot_off[h + 1];
    if (s1 - s0 <= kFixWarps) {
        // short split row: warp 0 sums its slots in order (k_spmm_fixup_warp's sum, so one
        // launch serves both kinds of split rows)
        if (w != 0 || lane >= G) return;
        float tot[1][E];
#pragma unroll
        for (int q = 0; q < E; q++) tot[0][q] = 0.f;
        for (int sl = s0; sl < s1; sl++) {
            const float* src = a.partial + ((int64_t)sl * WV + lane) * E;
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                const float4 p = *reinterpret_cast<const float4*>(src + q);
                tot[0][q] += p.x; tot[0][q + 1] += p.y; tot[0][q + 2] += p.z; tot[0][q + 3] += p.w;
            }
        }
        epilogue<T, 1>(a, r, a.out_compact ? h : r, lane, G, WV, tot);
        return;
    }
    float acc[E];
#pragma unroll
    for (int q = 0; q < E; q++) acc[q] = 0.f;
    if (lane < G) {
        for (int sl = s0 + w; sl < s1; sl += kFixWarps) {
            const float* src = a.partial + ((int64_t)sl * WV + lane) * E;
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                const float4 p = *reinterpret_cast<const float4*>(src + q);
                acc[q] += p.x; acc[q + 1] += p.y; acc[q + 2] += p.z; acc[q + 3] += p.w;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < E; q++) red[w][lane * E + q] = acc[q];
    __syncthreads();
    if (w == 0 && lane < G) {
        float tot[1][E];
#pragma unroll
        for (int q = 0; q < E; q++) {
            float t = 0.f;
            for (int k = 0; k < kFixWarps; k++) t += red[k][lane * E + q];
            tot[0][q] = t;
        }
        epilogue<T, 1>(a, r, a.out_compact ? h : r, lane, G, WV, tot);
    }
}

template <typename T, int R>
static grappa_status launch_grp(grappa_ctx* ctx, const SpmmArgs& a, int G, cudaStream_t s) {
    const int P = 32 / G;
    const int64_t vrows = a.n + a.n_slots;   // split-row segments first, then the rows
    if (vrows > 0) {
        const unsigned grid = (unsigned)ceil_div(ceil_div(vrows, P), 8);
        if (g_spmm_variant == 2) {
            if (a.col_scale || a.edge_w) k_spmm_grp<T, R, 8, true><<<grid, 256, 0, s>>>(a, G, P);
            else k_spmm_grp<T, R, 8, false><<<grid, 256, 0, s>>>(a, G, P);
        } else {
            if (a.col_scale || a.edge_w) k_spmm_grp<T, R, 4, true><<<grid, 256, 0, s>>>(a, G, P);
            else k_spmm_grp<T, R, 4, false><<<grid, 256, 0, s>>>(a, G, P);
        }
        GRAPPA_LAUNCHED(ctx);
    }
    if (a.n_heavy > 0) {
        k_spmm_fixup_blk<T><<<(unsigned)a.n_heavy, kFixWarps * 32, 0, s>>>(a, G);
        GRAPPA_LAUNCHED(ctx);
    }
    return GRAPPA_OK;
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

template <int R>
static grappa_status launch_grp16(grappa_ctx* ctx, const SpmmArgs& a, int G, cudaStream_t s) {
    const int P = 32 / G;
    const int64_t vrows = a.n + a.n_slots;
    if (vrows > 0) {
        k_spmm_grp16<R, 4><<<(unsigned)ceil_div(ceil_div(vrows, P), 8), 256, 0, s>>>(a, G, P);
        GRAPPA_LAUNCHED(ctx);
    }
    if (a.n_heavy > 0) {
        k_spmm_fixup_blk<__nv_bfloat16><<<(unsigned)a.n_heavy, kFixWarps * 32, 0, s>>>(a, 2 * G);
        GRAPPA_LAUNCHED(ctx);
    }
    return GRAPPA_OK;
}

template <typename T>
static grappa_status launch_t(grappa_ctx* ctx, const SpmmArgs& a, cudaStream_t s) {
    const int WV = a.width / Vec<T>::EPV;
    if (sizeof(T) == 2 && !a.col_scale && !a.edge_w && a.width % 16 == 0 && a.width / 16 <= 32 && g_spmm_variant == 0 &&
        g_wide_loads) {
        const int G16 = a.width / 16;
        if (G16 >= 16) return launch_grp16<1>(ctx, a, G16, s);
        if (G16 >= 8) return launch_grp16<2>(ctx, a, G16, s);
        if (G16 >= 4) return launch_grp16<4>(ctx, a, G16, s);
        return launch_grp16<8>(ctx, a, G16, s);
    }
    if (WV <= 32 && g_spmm_variant != 1) {
        // group-per-row kernel; R index registers per lane so a chunk holds >= 16 edges
        if (WV >= 16) return launch_grp<T, 1>(ctx, a, WV, s);
        if (WV >= 8) return launch_grp<T, 2>(ctx, a, WV, s);
        if (WV >= 4) return launch_grp<T, 4>(ctx, a, WV, s);
        return launch_grp<T, 8>(ctx, a, WV, s);
    }
    const int G = WV <= 32 ? WV : 32;
    const int P = 32 / G;
    const int cpl = (WV + G - 1) / G;
    if (cpl <= 1) return launch_cpl<T, 1>(ctx, a, G, P, s);
    if (cpl <= 2) return launch_cpl<T, 2>(ctx, a, G, P, s);
    if (cpl <= 4) return launch_cpl<T, 4>(ctx, a, G, P, s);
    if (cpl <= 8) return launch_cpl<T, 8>(ctx, a, G, P, s);
    if (cpl <= 12) return launch_cpl<T, 12>(ctx, a, G, P, s);
    set_error("spmm: width %d too large", a.width);
    return GRAPPA_E_SHAPE;
}

// ------------------------------------------------------------------ fused aggregate -> transform
// k_spmm_mm: persistent, one 1024-thread CTA per SM.  Per 128-row tile (rows in the
// degree-bucketed order, split rows first -- their aggregates come pre-combined from the
// segment pre-pass in `hagg`):
//   1. the 32 warps gather-accumulate the tile's rows (grp_accumulate, fp32), apply self /
//      row scale, round to bf16 and write them straight into shared memory in the UMMA K-major
//      SWIZZLE_128B layout (and to agg_out if asked);
//   2. one thread issues K/16 tcgen05.mma (A = that tile, B = the weights, converted to bf16
//      once per CTA and resident in smem) into one of two TMEM accumulators;
//   3. while those MMAs run, all warps drain the PREVIOUS tile's accumulator (tcgen05.ld ->
//      relu / relu'-gate -> bf16 -> global rows).
// The transform costs no HBM traffic of its own: the n x K aggregate never leaves the SM.
constexpr int kMMWarps = 32;
constexpr int kMMTile = 128;
constexpr int kMMMaxSmem = 227 * 1024;
// off by default: measured slower than SpMM + tcgen05 GEMM on products;
// kept selectable ("fuse" = 1) and parity-tested
static int g_fuse_variant = 0;
void spmm_set_fuse(int v) { g_fuse_variant = v; }

struct AggMM {
    int64_t n, n_heavy;
    int num_tiles, K, kbt, N, b_trans, relu, self;
    const int64_t* rowptr;
    const int32_t* col;
    const int32_t* row_order;
    const int32_t* heavy_rows;
    const __nv_bfloat16* hagg;
    const __nv_bfloat16* X;
    const float* rs;
    const float* cs;
    const float* W;
    const __nv_bfloat16* mask;
    __nv_bfloat16* out;
    __nv_bfloat16* agg_out;
    uint32_t tmem_cols;
};

static size_t mm_smem(int kbt, int N) {
    return 1024 + (size_t)kbt * kMMTile * 128 + (size_t)kbt * N * 128 + 2 * kMMTile * 4 + 64;
}

template <int R>
__global__ void __launch_bounds__(kMMWarps * 32, 1) k_spmm_mm(AggMM p, int G, int P) {
    using T = __nv_bfloat16;
    constexpr int E = 8;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;                                           // kbt x [128 rows x 128 B]
    uint8_t* sB = sA + (size_t)p.kbt * kMMTile * 128;             // kbt x [N rows x 128 B]
    int32_t* srow = (int32_t*)(sB + (size_t)p.kbt * p.N * 128);   // [2][128] tile rows
    uint64_t* done = (uint64_t*)(srow + 2 * kMMTile);
    uint32_t* tmem_slot = (uint32_t*)(done + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // weights -> smem once: bf16, K-major SWIZZLE_128B (B operand = N rows of K), zero padded
    const int nchunks = p.kbt * p.N * 8;
    for (int idx = threadIdx.x; idx < nchunks; idx += blockDim.x) {
        const int kb = idx / (p.N * 8), rem = idx % (p.N * 8), n = rem >> 3, ch = rem & 7;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int k = kb * 64 + ch * 8 + q;
            float f = 0.f;
            if (k < p.K) f = p.b_trans ? p.W[(int64_t)n * p.K + k] : p.W[(int64_t)k * p.N + n];
            v[q] = __float2bfloat16_rn(f);
        }
        *reinterpret_cast<uint4*>(sB + (size_t)kb * p.N * 128 + tc::sw128_off(n, ch)) =
            *reinterpret_cast<const uint4*>(v);
    }
    if (threadIdx.x == 0) {
        tc::mbar_init(&done[0], 1);
        tc::mbar_init(&done[1], 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, p.tmem_cols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = tc::idesc_bf16(kMMTile, p.N, 0, 0);
    const int slot = lane / G, sub = lane - slot * G;
    const int q4 = warp & 3, cg = warp >> 2;       // epilogue: TMEM lane quarter, column group

    int it = 0;
    for (int tile = blockIdx.x;; tile += gridDim.x, it++) {
        const bool have = tile < p.num_tiles;
        const int buf = it & 1;
        if (have) {
            for (int base = warp * P; base < kMMTile; base += kMMWarps * P) {
                const int tr = base + slot;
                const int64_t vi = (int64_t)tile * kMMTile + tr;
                int64_t v = -1, e0 = 0;
                int deg = 0;
                bool heavy = false;
                if (slot < P && tr < kMMTile && vi < p.n) {
                    if (vi < p.n_heavy) {
                        v = p.heavy_rows[vi];
                        heavy = true;
                    } else {
                        v = p.row_order[vi];
                        e0 = p.rowptr[v];
                        deg = (int)(p.rowptr[v + 1] - e0);
                    }
                }
                float acc[E];
#pragma unroll
                for (int q = 0; q < E; q++) acc[q] = 0.f;
                if (p.cs) grp_accumulate<T, R, 4, true>(p.X, p.col, p.cs, e0, deg, G, slot, sub, acc);
                else grp_accumulate<T, R, 4, false>(p.X, p.col, p.cs, e0, deg, G, slot, sub, acc);
                if (v >= 0) {
                    uint4 pk;
                    if (heavy) {
                        pk = *reinterpret_cast<const uint4*>(p.hagg + (vi * p.K + sub * E));
                    } else {
                        // same order as spmm's epilogue: (acc + cs_v x_v) * rs_v
                        if (p.self) {
                            float f[E];
                            Vec<T>::to_f(Vec<T>::load(p.X + ((int64_t)v * p.K + sub * E)), f);
                            const float c = p.cs ? p.cs[v] : 1.f;
#pragma unroll
                            for (int q = 0; q < E; q++) acc[q] = fmaf(c, f[q], acc[q]);
                        }
                        const float r = p.rs ? p.rs[v] : 1.f;
                        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * q] * r, acc[2 * q + 1] * r);
                            w[q] = *reinterpret_cast<uint32_t*>(&b);
                        }
                    }
                    *reinterpret_cast<uint4*>(sA + (sub >> 3) * (kMMTile * 128) + tc::sw128_off(tr, sub & 7)) = pk;
                    if (p.agg_out) *reinterpret_cast<uint4*>(p.agg_out + (v * p.K + sub * E)) = pk;
                    if (sub == 0) srow[buf * kMMTile + tr] = (int32_t)v;
                } else if (slot < P && tr < kMMTile && sub == 0) {
                    srow[buf * kMMTile + tr] = -1;
                }
            }
            tc::fence_proxy_async();                 // staged rows -> visible to the tensor core
        }
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (have && threadIdx.x == 0) {
            const uint32_t d = tmem + (uint32_t)(buf * p.N);
            const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
            for (int ks = 0; ks < p.K / 16; ks++) {
                const int kb = ks >> 2, k = ks & 3;
                tc::mma_f16(d, tc::smem_desc_sw128(a0 + kb * (kMMTile * 128) + k * 32, 0, 1024),
                            tc::smem_desc_sw128(b0 + kb * p.N * 128 + k * 32, 0, 1024), idesc, ks > 0);
            }
            tc::mma_commit(&done[buf]);
        }
        if (it > 0) {
            // epilogue of the previous tile (its MMAs completed before this iteration began)
            const int pb = buf ^ 1;
            const int tr = q4 * 32 + lane;
            const int64_t v = srow[pb * kMMTile + tr];
            const uint32_t tb = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(pb * p.N);
            for (int c0 = cg * 16; c0 < p.N; c0 += (kMMWarps / 4) * 16) {
                float x[16];
                tc::tmem_ld16(tb + c0, x);
                if (v < 0) continue;
                if (p.mask) {
                    __align__(16) __nv_bfloat16 mk[16];
                    const uint4* src = reinterpret_cast<const uint4*>(p.mask + (v * p.N + c0));
                    reinterpret_cast<uint4*>(mk)[0] = __ldg(src);
                    reinterpret_cast<uint4*>(mk)[1] = __ldg(src + 1);
#pragma unroll
                    for (int i = 0; i < 16; i++) x[i] = __bfloat162float(mk[i]) > 0.f ? x[i] : 0.f;
                }
                if (p.relu) {
#pragma unroll
                    for (int i = 0; i < 16; i++) x[i] = fmaxf(x[i], 0.f);
                }
                __align__(16) __nv_bfloat16 o[16];
#pragma unroll
                for (int i = 0; i < 16; i++) o[i] = __float2bfloat16_rn(x[i]);
                uint4* dst = reinterpret_cast<uint4*>(p.out + (v * p.N + c0));
                dst[0] = reinterpret_cast<const uint4*>(o)[0];
                dst[1] = reinterpret_cast<const uint4*>(o)[1];
            }
        }
        if (!have) break;
        tc::mbar_wait(&done[buf], (uint32_t)((it >> 1) & 1));   // sA free, accumulator ready
        tc::fence_after();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, p.tmem_cols);
    }
}

bool spmm_mm_supported(const grappa_part* part, int K, int N, grappa_dtype dt) {
    const int kbt = (int)ceil_div(K, 64);
    return g_fuse_variant == 1 && g_spmm_variant == 0 && dt == GRAPPA_BF16 && K % 16 == 0 &&
           N % 16 == 0 && K >= 16 && K <= 256 && N >= 16 && N <= 256 && part->row_order.p != nullptr &&
           part->info.n_core < (1ll << 31) && mm_smem(kbt, N) <= (size_t)kMMMaxSmem;
}

template <int R>
static void launch_mm(const AggMM& p, int G, size_t smem, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_spmm_mm<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMMMaxSmem);
        attr = true;
    }
    k_spmm_mm<R><<<grid, kMMWarps * 32, smem, s>>>(p, G, 32 / G);
}

grappa_status spmm_mm(grappa_ctx* ctx, const grappa_part* part, const AggMMArgs& m, cudaStream_t s) {
    const grappa_part_info& I = part->info;
    if (!spmm_mm_supported(part, m.K, m.N, GRAPPA_BF16)) {
        set_error("spmm_mm: unsupported K=%d N=%d", m.K, m.N);
        return GRAPPA_E_SUPPORT;
    }
    const double K = m.K, N = m.N, nnz = (double)I.nnz, n = (double)I.n_core;
    const double per_edge = 4.0 + (m.col_scale ? 4.0 : 0.0) + 2.0 * K;
    const double per_row = 8.0 + (m.row_scale ? 4.0 : 0.0) + (m.col_scale ? 4.0 : 0.0) +
                           (m.self ? 2.0 * K : 0.0) + 2.0 * N + (m.mask ? 2.0 * N : 0.0) +
                           (m.agg_out ? 2.0 * K : 0.0);
    ProfScope ps(ctx, s, GRAPPA_K_SPMM, nnz * per_edge + n * per_row + 4.0 * K * N,
                 2.0 * nnz * K + 2.0 * n * K * N);
    if (I.n_core == 0) return GRAPPA_OK;
    if (I.n_heavy > 0) {
        // split rows: segment partials + in-order combine -> hagg[h] (no activation)
        SpmmArgs a;
        a.n = 0;                              // segments only
        a.nnz = I.nnz;
        a.rowptr = I.rowptr;
        a.col = I.col;
        a.n_slots = I.n_slots;
        a.n_heavy = I.n_heavy;
        a.slot_row = (const int32_t*)part->slot_row.p;
        a.slot_seg = (const int32_t*)part->slot_seg.p;
        a.heavy_rows = (const int32_t*)part->heavy_rows.p;
        a.heavy_slot_off = (const int32_t*)part->heavy_slot_off.p;
        a.X = m.X; a.width = m.K; a.row_scale = m.row_scale; a.col_scale = m.col_scale;
        a.self = m.self; a.out = m.hagg; a.out_compact = 1; a.partial = m.partial;
        GRAPPA_TRY(launch_t<__nv_bfloat16>(ctx, a, s));
    }
    AggMM p;
    p.n = I.n_core; p.n_heavy = I.n_heavy;
    p.num_tiles = (int)ceil_div(I.n_core, kMMTile);
    p.K = m.K; p.kbt = (int)ceil_div(m.K, 64); p.N = m.N;
    p.b_trans = m.b_trans; p.relu = m.relu; p.self = m.self;
    p.rowptr = I.rowptr; p.col = I.col;
    p.row_order = (const int32_t*)part->row_order.p;
    p.heavy_rows = (const int32_t*)part->heavy_rows.p;
    p.hagg = (const __nv_bfloat16*)m.hagg;
    p.X = (const __nv_bfloat16*)m.X;
    p.rs = m.row_scale; p.cs = m.col_scale; p.W = m.W;
    p.mask = (const __nv_bfloat16*)m.mask;
    p.out = (__nv_bfloat16*)m.out;
    p.agg_out = (__nv_bfloat16*)m.agg_out;
    uint32_t cols = 32;
    while ((int)cols < 2 * m.N) cols <<= 1;
    p.tmem_cols = cols;
    // >= 116 KB of shared memory keeps it at one CTA per SM (the CTA owns 2N TMEM columns)
    const size_t smem = std::max<size_t>(mm_smem(p.kbt, m.N), 116 * 1024);
    const int grid = (int)std::min<int64_t>(p.num_tiles, ctx->sm_count);
    const int G = m.K / 8;
    if (G >= 16) launch_mm<1>(p, G, smem, grid, s);
    else if (G >= 8) launch_mm<2>(p, G, smem, grid, s);
    else if (G >= 4) launch_mm<4>(p, G, smem, grid, s);
    else launch_mm<8>(p, G, smem, grid, s);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

grappa_status spmm(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                   cudaStream_t s) {
    const grappa_part_info& I = part->info;
    a.n = I.n_core;
    a.nnz = I.nnz;
    a.rowptr = I.rowptr;
    a.col = I.col;
    a.n_slots = I.n_slots;
    a.n_heavy = I.n_heavy;
    a.slot_row = (const int32_t*)part->slot_row.p;
    a.slot_seg = (const int32_t*)part->slot_seg.p;
    a.heavy_rows = (const int32_t*)part->heavy_rows.p;
    a.heavy_slot_off = (const int32_t*)part->heavy_slot_off.p;
    a.row_order = g_spmm_variant == 3 ? nullptr : (const int32_t*)part->row_order.p;
    a.row_desc = g_spmm_variant == 3 ? nullptr : (const int4*)part->row_desc.p;
    return spmm_csr(ctx, a, dt, s);
}

grappa_status spmm_t(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                     cudaStream_t s) {
    if (!part->halo) return spmm(ctx, part, a, dt, s);     // induced-core: A^T = A
    const grappa_part_info& I = part->info;
    a.n = I.n_core;
    a.nnz = I.nnz;
    a.rowptr = (const int64_t*)part->t_rowptr.p;
    a.col = (const int32_t*)part->t_col.p;
    a.n_slots = part->t_n_slots;
    a.n_heavy = part->t_n_heavy;
    a.slot_row = (const int32_t*)part->t_slot_row.p;
    a.slot_seg = (const int32_t*)part->t_slot_seg.p;
    a.heavy_rows = (const int32_t*)part->t_heavy_rows.p;
    a.heavy_slot_off = (const int32_t*)part->t_heavy_slot_off.p;
    a.row_order = g_spmm_variant == 3 ? nullptr : (const int32_t*)part->t_row_order.p;
    a.row_desc = g_spmm_variant == 3 ? nullptr : (const int4*)part->t_row_desc.p;
    return spmm_csr(ctx, a, dt, s);
}

grappa_status spmm_csr(grappa_ctx* ctx, SpmmArgs a, grappa_dtype dt, cudaStream_t s) {
    if (a.width % 8 != 0) {
        set_error("spmm: width %d not a multiple of 8", a.width);
        return GRAPPA_E_SHAPE;
    }
    struct { int64_t n_core, nnz; } I{a.n, a.nnz};
    const double es = dt == GRAPPA_BF16 ? 2.0 : 4.0, w = a.width, nnz = (double)I.nnz;
    const double per_edge = 4.0 + (a.col_scale || a.edge_w ? 4.0 : 0.0) + w * es;
    const bool self_coef = a.self && (a.self_sep ? a.self_scale != nullptr : a.col_scale != nullptr);
    const double per_row = 8.0 + (a.row_scale ? 4.0 : 0.0) + (self_coef ? 4.0 : 0.0) +
                           (a.nbr_scale ? 4.0 : 0.0) + (a.self ? w * es : 0.0) + w * es +
                           (a.accumulate ? w * es : 0.0) + (a.mask ? w * es : 0.0);
    ProfScope ps(ctx, s, GRAPPA_K_SPMM, nnz * per_edge + (double)I.n_core * per_row, 2.0 * nnz * w);
    return dt == GRAPPA_BF16 ? launch_t<__nv_bfloat16>(ctx, a, s) : launch_t<float>(ctx, a, s);
}

}  // namespace grappa
