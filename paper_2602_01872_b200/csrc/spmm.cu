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
// dispatch knob (tests / A-B timing) for narrow rows: 0 = row-group kernel, unweighted gathers
// through grp_accumulate_lean (default; measured best), 1 = warp-per-row kernel, 2 = row-group
// kernel with 8 loads in flight (more registers, fewer resident warps: slower on B200),
// 3 = row-group kernel over the rows in natural order (no degree bucketing), 4 = TMA row gather
// (spmm_tma.cu), 5 = row-group kernel with the previous unweighted schedule (grp_accumulate).
// Measured and not kept: a persistent grid-stride version of the lean kernel (255 vs 220 us per
// products call: static row-group assignment loses the block scheduler's balancing) and a
// packed epilogue (FMUL2 / FFMA2, ReLU folded into the bf16 pack) with a division-free slot
// split (242 vs 220 us: more live registers, spills at the 32-register bound); a warp-per-
// split-row fix-up, 8 rows per block (the call 220 -> 241 us: a hub's 100+ segments summed by one
// warp became the tail); the split-row
// combine fused into this kernel (last-arriving segment sums its row; 436 us: the fence and
// counter path inflated every launch); a tensor-core aggregation (8 targets per warp, their edge
// lists walked 16 at a time, neighbour rows staged by cp.async, D += S^T B with B the 0/1
// edge-to-target matrix via ldmatrix.trans + mma.sync m16n8k16; correct to 1e-6) at 506 us:
// latency-bound on the staged chunk, ~2.3x slower at equal bytes in flight; the row's own
// vector and row scale requested before the gathers (244 vs 222 us: spills at 32 registers).
static inline int spmm_var(const grappa_ctx* c) { return c ? c->var_spmm : 0; }

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
    const T* X = reinterpret_cast<const T*>(a.X_self ? a.X_self : a.X);   // the self term's rows
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
        if (a.accumulate && v < a.acc_rows) {
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
    // unweighted gathers: row s of this lane's 16-byte column at base_lane + s * row bytes (one
    // IMAD.WIDE.U32 per gathered vector instead of the signed 64-bit index arithmetic)
    const uint64_t base_lane = reinterpret_cast<uint64_t>(X) + (uint64_t)sub * 16;
    const uint32_t rowb = (uint32_t)WV * 16;
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
                                      : Vec<T>::load_ordered(reinterpret_cast<const T*>(
                                            base_lane + (uint64_t)(uint32_t)s * rowb));
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

// Predicated gather-add of one 16-byte vector: `ok` guards both the load and the adds, so a
// masked-off edge costs neither a zeroing move nor a wasted add (ISETP once, shared by both).
__device__ __forceinline__ void pred_gather_add(float (&acc)[8], const __nv_bfloat16* p, bool ok) {
    uint32_t x0, x1, x2, x3;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                 "@q ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%5];\n\t}"
                 : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"((int)ok), "l"(p));
    asm volatile("{\n\t.reg .pred q;\n\t.reg .b16 l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
                 "setp.ne.b32 q, %12, 0;\n\t"
                 "mov.b32 {l0, h0}, %8;\n\tmov.b32 {l1, h1}, %9;\n\t"
                 "mov.b32 {l2, h2}, %10;\n\tmov.b32 {l3, h3}, %11;\n\t"
                 "@q add.rn.f32.bf16 %0, l0, %0;\n\t@q add.rn.f32.bf16 %1, h0, %1;\n\t"
                 "@q add.rn.f32.bf16 %2, l1, %2;\n\t@q add.rn.f32.bf16 %3, h1, %3;\n\t"
                 "@q add.rn.f32.bf16 %4, l2, %4;\n\t@q add.rn.f32.bf16 %5, h2, %5;\n\t"
                 "@q add.rn.f32.bf16 %6, l3, %6;\n\t@q add.rn.f32.bf16 %7, h3, %7;\n\t}"
                 : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]),
                   "+f"(acc[6]), "+f"(acc[7])
                 : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"((int)ok));
}
__device__ __forceinline__ void pred_gather_add(float (&acc)[4], const float* p, bool ok) {
    if (ok) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
    }
}

// Unweighted gather-accumulate (every GCN call after R29, SAGE forward): same rows, lanes and
// summation order as grp_accumulate<.., false> (bitwise the same sums), but the edges of a
// G-edge sub-chunk are walked in groups of UL with compile-time offsets and one predicate per
// edge that guards both the load and its adds, and the next sub-chunk's column index is loaded
// while this one is gathered: a gathered vector costs a shuffle, a compare, an IMAD.WIDE, the
// load and its 8 adds (~14 issue slots) instead of ~20-24 (per-edge lane / bound arithmetic,
// selects, zeroing moves; the kernel is issue-bound).  Measured on a products partition (bf16
// 128 wide): 346 -> 222 us per call with UL = 2 at 32 registers (UL = 1: 247, 3: 237, UL = 4 at
// 40 registers: 240; the whole 32-edge sub-chunk unrolled spilled).
template <typename T, int UL>
__device__ __forceinline__ void grp_accumulate_lean(const T* __restrict__ X, const int32_t* __restrict__ col,
                                                    int64_t e0, int deg, int G, int slot, int sub,
                                                    float (&acc)[Vec<T>::EPV]) {
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    const uint64_t base_lane = reinterpret_cast<uint64_t>(X) + (uint64_t)sub * 16;
    const uint32_t rowb = (uint32_t)G * 16;
    const int slotG = slot * G;
    const int32_t* cl = col + e0 + sub;
    int idx = sub < deg ? __ldg(cl) : 0;
    for (int off = 0; off < maxdeg; off += G) {
        // the next sub-chunk's index is in flight while this one's rows are gathered
        const int nidx = off + G + sub < deg ? __ldg(cl + off + G) : 0;
        const int jmax = min(G, maxdeg - off);          // warp-uniform
        const int rem = min(G, deg - off);              // this lane's valid edges here
#pragma unroll 1
        for (int jb = 0; jb < jmax; jb += UL) {
            const int lb = slotG + jb, rb = rem - jb;
#pragma unroll
            for (int u = 0; u < UL; u++) {
                const uint32_t s = (uint32_t)__shfl_sync(0xffffffffu, idx, lb + u);
                pred_gather_add(acc, reinterpret_cast<const T*>(base_lane + (uint64_t)s * rowb), u < rb);
            }
        }
        idx = nidx;
    }
}

// Narrow rows: every group of G = W/EPV lanes owns a different row, so a warp carries
// P = 32/G independent rows and their dependent load chains (rowptr -> col -> scale /
// feature row) overlap; no cross-group reduction is needed.
template <typename T, int R, int U, bool WT, bool LEAN = false, int MB = 1>
__global__ void __launch_bounds__(256, MB) k_spmm_grp(SpmmArgs a, int G, int P, unsigned gmagic) {
    constexpr int E = Vec<T>::EPV;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // lane / G without an integer division (lane < 32, G <= 32): lane * gmagic >> 16 with
    // gmagic = ceil(2^16 / G) (host) is exact, the rounding term is below 32 / 2^16
    const int slot = (int)(((unsigned)lane * gmagic) >> 16), sub = lane - slot * G;
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
    if (LEAN)
        grp_accumulate_lean<T, U>(reinterpret_cast<const T*>(a.X), a.col, e0, (int)(e1 - e0), G, slot,
                                  sub, acc);
    else
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
        const unsigned gm = (65536u + (unsigned)G - 1u) / (unsigned)G;
        if (spmm_var(ctx) == 2) {
            if (a.col_scale || a.edge_w) k_spmm_grp<T, R, 8, true><<<grid, 256, 0, s>>>(a, G, P, gm);
            else k_spmm_grp<T, R, 8, false><<<grid, 256, 0, s>>>(a, G, P, gm);
        } else {
            // weighted gathers keep grp_accumulate: a lean weighted walk (weight loaded one
            // sub-chunk ahead and shuffled with the index, predicated FFMA2) measured no faster
            // (GCN input layer 378 -> 402 us per products call; node-level epoch 41.7 -> 42.4 ms)
            if (a.col_scale || a.edge_w) k_spmm_grp<T, R, 4, true><<<grid, 256, 0, s>>>(a, G, P, gm);
            else if (spmm_var(ctx) == 5) k_spmm_grp<T, R, 4, false><<<grid, 256, 0, s>>>(a, G, P, gm);
            else k_spmm_grp<T, R, 2, false, true, 8><<<grid, 256, 0, s>>>(a, G, P, gm);
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

template <typename T>
static grappa_status launch_t(grappa_ctx* ctx, const SpmmArgs& a, cudaStream_t s) {
    const int WV = a.width / Vec<T>::EPV;
    if (WV <= 32 && spmm_var(ctx) != 1) {
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

// split-row combine for bf16 rows (the TMA kernel's fix-up: same launch as launch_grp's)
grappa_status spmm_fixup(grappa_ctx* ctx, const SpmmArgs& a, cudaStream_t s) {
    if (a.n_heavy > 0) {
        k_spmm_fixup_blk<__nv_bfloat16><<<(unsigned)a.n_heavy, kFixWarps * 32, 0, s>>>(a, a.width / 8);
        GRAPPA_LAUNCHED(ctx);
    }
    return GRAPPA_OK;
}

// out[v] = scale[v] * X[v] (rounded to the storage dtype), 16 bytes per thread: the GCN input
// layer's source normalisation applied once per row, so its aggregation gathers unweighted rows
// (R29c) instead of loading scale[u] per edge (the weighted walk: 378 us per products call at
// width 112, the unweighted one ~205 us + this pass ~45 us)
template <typename T>
__global__ void k_row_scale(int64_t n, int wv, const T* __restrict__ X, const float* __restrict__ scale,
                            T* __restrict__ out) {
    constexpr int E = Vec<T>::EPV;
    const int64_t total = n * wv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / wv;
        const float sc = __ldg(scale + v);
        float f[E];
        Vec<T>::to_f(Vec<T>::load(X + i * E), f);
#pragma unroll
        for (int q = 0; q < E; q++) f[q] *= sc;
        Vec<T>::store(out + i * E, f);
    }
}

grappa_status row_scale(grappa_ctx* ctx, const void* X, int64_t n, int width, const float* scale, void* out,
                        grappa_dtype dt, cudaStream_t s) {
    if (n <= 0) return GRAPPA_OK;
    const int E = dt == GRAPPA_BF16 ? 8 : 4;
    const int wv = width / E;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n * wv, 256), (int64_t)ctx->sm_count * 16);
    if (dt == GRAPPA_BF16)
        k_row_scale<__nv_bfloat16><<<grid, 256, 0, s>>>(n, wv, (const __nv_bfloat16*)X, scale, (__nv_bfloat16*)out);
    else
        k_row_scale<float><<<grid, 256, 0, s>>>(n, wv, (const float*)X, scale, (float*)out);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

static double spmm_bytes(const SpmmArgs& a, grappa_dtype dt) {
    const double es = dt == GRAPPA_BF16 ? 2.0 : 4.0, w = a.width, nnz = (double)a.nnz;
    const double per_edge = 4.0 + (a.col_scale || a.edge_w ? 4.0 : 0.0) + w * es;
    const bool self_coef = a.self && (a.self_sep ? a.self_scale != nullptr : a.col_scale != nullptr);
    const double per_row = 8.0 + (a.row_scale ? 4.0 : 0.0) + (self_coef ? 4.0 : 0.0) +
                           (a.nbr_scale ? 4.0 : 0.0) + (a.self ? w * es : 0.0) + w * es +
                           (a.accumulate ? w * es : 0.0) + (a.mask ? w * es : 0.0);
    return nnz * per_edge + (double)a.n * per_row;
}

// a partition operator: the TMA-gather kernel when selected and applicable (spmm_tma.cu), else
// the row-group / warp-per-row kernels
static grappa_status spmm_part(grappa_ctx* ctx, const grappa_part* part, bool transpose, SpmmArgs& a,
                               grappa_dtype dt, cudaStream_t s) {
    if (a.width % 8 != 0) {
        set_error("spmm: width %d not a multiple of 8", a.width);
        return GRAPPA_E_SHAPE;
    }
    ProfScope ps(ctx, s, GRAPPA_K_SPMM, spmm_bytes(a, dt), 2.0 * (double)a.nnz * a.width);
    if (spmm_tma_eligible(ctx, a, dt)) return spmm_tma(ctx, part, transpose, a, s);
    return dt == GRAPPA_BF16 ? launch_t<__nv_bfloat16>(ctx, a, s) : launch_t<float>(ctx, a, s);
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
    a.row_order = spmm_var(ctx) == 3 ? nullptr : (const int32_t*)part->row_order.p;
    a.row_desc = spmm_var(ctx) == 3 ? nullptr : (const int4*)part->row_desc.p;
    return spmm_part(ctx, part, false, a, dt, s);
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
    a.row_order = spmm_var(ctx) == 3 ? nullptr : (const int32_t*)part->t_row_order.p;
    a.row_desc = spmm_var(ctx) == 3 ? nullptr : (const int4*)part->t_row_desc.p;
    return spmm_part(ctx, part, true, a, dt, s);
}

grappa_status spmm_csr(grappa_ctx* ctx, SpmmArgs a, grappa_dtype dt, cudaStream_t s) {
    if (a.width % 8 != 0) {
        set_error("spmm: width %d not a multiple of 8", a.width);
        return GRAPPA_E_SHAPE;
    }
    ProfScope ps(ctx, s, GRAPPA_K_SPMM, spmm_bytes(a, dt), 2.0 * (double)a.nnz * a.width);
    return dt == GRAPPA_BF16 ? launch_t<__nv_bfloat16>(ctx, a, s) : launch_t<float>(ctx, a, s);
}

}  // namespace grappa
