// spmm_tma.cu -- the partition-local aggregation (SpMM of a4/a6) with TMA row gathers.
//
// PAPER: P:141/P:177 (§3.2 isolated message passing over local nodes and edges only),
// P:435-437 (§5.1 GCN aggregation); north_star "warp-per-row, vectorised, coalesced
// CSR gather-sum SpMM with shared-memory/TMA staging of feature tiles".
//
//   out[v] = act( rs[v] * ( self * X[v] + ns[v] * sum_{u in N_loc(v)} X[u] ) )      (bf16 rows)
//   split-row segments: partial[k] = sum over the segment's edges (fp32), combined in segment
//   order by k_spmm_fixup_blk (spmm.cu) -- the row-group kernel's arithmetic, bit for bit.
//
// Why: the row-group kernel (spmm.cu) spends ~22 instructions per gathered 16-byte vector
// (shuffle, 64-bit address, predicates, 8 adds) and holds only 2 gathers in flight per lane at
// 32 registers; it runs at ~55% of the L2 row-gather ceiling, issue-bound.  Here the gathers
// leave the SM's instruction stream: one producer warp issues cp.async.bulk.tensor ...
// tile::gather4 (4 whole rows per instruction) into a shared-memory ring, from a gather-index
// stream precomputed per partition (the plan), and 8 consumer warps only read shared memory
// and add (1 LDS.128 + 8 FHADD per 16-byte vector).  Bytes in flight are bounded by the ring
// (160 KB per SM), not by registers.
//
// Plan (tma_plan_build): the SpMM's row space -- split-row segments (slots) first, then the
// non-split rows in the degree-bucketed order (descending degree) -- is cut into 16-row tiles;
// tile t goes to CTA t mod grid (degree-interleaved load balance); tiles are stored CTA-major so
// every CTA owns ONE contiguous range of steps of the index stream.  Tile with row degrees
// d_0..d_15 has 1 + max d steps: step 0 gathers each row's own row (the self term), step j >= 1
// the (j-1)-th neighbour (a row with fewer neighbours gathers its own row again and ignores
// it).  Rows are processed in the same edge order as the row-group kernel, so the fp32 sums
// are bitwise the same.
//
// Kernel: persistent, one CTA (9 warps) per SM.  The producer cuts the CTA's step range into
// chunks of <= 8 steps (16 rows x 8 steps x 2W bytes), places each chunk contiguously in a
// 160 KB byte ring (chunks freed in order), and per chunk: arrive.expect_tx on the chunk slot's
// full barrier, then one gather4 per lane (lane l = step l/4, rows 4(l%4)..+3).  Consumer warp w
// owns tile rows 2w, 2w+1 (G = W/8 lanes per row, one 16-byte vector each); it walks the steps
// in order, keeps the self vector, accumulates neighbour vectors into 8 fp32 registers, and at
// a tile's last step writes the row (bf16) or the segment partial (fp32).  One empty-barrier
// arrival per consumer warp per chunk.
#include "part.cuh"
#include "scan.cuh"
#include "spmm.cuh"
#include "tc.cuh"

namespace grappa {

grappa_status tma_map_rows_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int cols);

namespace {

constexpr int kTR = 16;                 // rows per tile
constexpr int kCW = 8;                  // consumer warps (2 tile rows each)
// producer warps: a warp issues its gather4s one lane at a time (the row ids move to uniform
// registers per instruction, ~90 cycles each), so one warp feeds ~2.6 TB/s; 6 warps, each
// filling whole chunks round-robin, measured ~15 TB/s on L2-resident rows (scripts/probe/g4bw.cu)
constexpr int kPW = 6;
constexpr int kThreads = (kCW + kPW) * 32;
constexpr int kSPC = 4;                 // steps per chunk: 4 x 4 gather4 (16 producer lanes)
constexpr int kNSlot = 16;              // max chunk slots (full / empty barrier pairs)
constexpr int kRing = 176 * 1024;       // gather ring bytes (chunk-sized slots)
constexpr int kSmem = kRing + 2 * kNSlot * 8 + 64;
constexpr uint32_t kSlotFlag = 0x80000000u;

struct PlanSrc {
    int64_t V, n_slots, n_heavy, T;      // row space = slots + non-split rows; T tiles
    const int64_t* rowptr;
    const int32_t* slot_row;
    const int32_t* slot_seg;
    const int4* row_desc;                // {v, deg, e0 lo, e0 hi}, split rows first (n_heavy)
    const int32_t* col;
    int grid;
    int64_t tpc;
};

// descriptor of row-space entry i: output (row id, or slot id | flag), degree, first edge, own row
__device__ __forceinline__ void vrow_desc(const PlanSrc& p, int64_t i, uint32_t& out, int32_t& deg, int64_t& e0,
                                          int32_t& self_row) {
    if (i < p.n_slots) {
        const int32_t r = p.slot_row[i], sg = p.slot_seg[i];
        const int64_t a = p.rowptr[r] + (int64_t)sg * kSegLen;
        const int64_t b = min(p.rowptr[r + 1], a + kSegLen);
        out = (uint32_t)i | kSlotFlag;
        deg = (int32_t)(b - a);
        e0 = a;
        self_row = r;
    } else {
        const int4 d = p.row_desc[p.n_heavy + (i - p.n_slots)];
        out = (uint32_t)d.x;
        deg = d.y;
        e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
        self_row = d.x;
    }
}

// CTA-major tile slot q -> original tile (tile t runs on CTA t mod grid)
__device__ __forceinline__ int64_t orig_tile(const PlanSrc& p, int64_t q) {
    const int64_t b = q / p.tpc, k = q - b * p.tpc;
    return k * p.grid + b;
}

__global__ void k_tma_tile_steps(PlanSrc p, int32_t* __restrict__ tsteps) {
    const int64_t nq = (int64_t)p.grid * p.tpc;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = orig_tile(p, q);
        int32_t steps = 0;
        if (t < p.T) {
            int32_t dmax = 0;
            for (int r = 0; r < kTR; r++) {
                const int64_t i = t * kTR + r;
                if (i >= p.V) break;
                uint32_t out; int32_t deg, self_row; int64_t e0;
                vrow_desc(p, i, out, deg, e0, self_row);
                dmax = max(dmax, deg);
            }
            steps = dmax + 1;
        }
        tsteps[q] = steps;
    }
}

// thread per (tile slot, row): the row's info and its column of the index stream
__global__ void k_tma_fill(PlanSrc p, const int32_t* __restrict__ tsteps, const int64_t* __restrict__ toff,
                           int2* __restrict__ tinfo, int32_t* __restrict__ stream) {
    const int64_t n = (int64_t)p.grid * p.tpc * kTR;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = x / kTR;
        const int r = (int)(x - q * kTR);
        const int32_t steps = tsteps[q];
        const int64_t t = orig_tile(p, q);
        const int64_t i = t * kTR + r;
        int32_t* dst = stream + toff[q] * kTR + r;
        if (t < p.T && i < p.V) {
            uint32_t out; int32_t deg, self_row; int64_t e0;
            vrow_desc(p, i, out, deg, e0, self_row);
            tinfo[x] = make_int2((int)out, deg);
            dst[0] = self_row;
            for (int32_t j = 1; j < steps; j++) dst[(int64_t)j * kTR] = j - 1 < deg ? p.col[e0 + j - 1] : self_row;
        } else {
            tinfo[x] = make_int2(-1, -1);
            for (int32_t j = 0; j < steps; j++) dst[(int64_t)j * kTR] = 0;
        }
    }
}

struct TsRead {
    const int32_t* a;
    __device__ int32_t operator()(int64_t i) const { return a[i]; }
};
struct TsWrite {
    int64_t* out;
    __device__ void operator()(int64_t i, int64_t p, int32_t) const { out[i] = p; }
    __device__ void finish(int64_t n, int64_t total) const { out[n] = total; }
};

struct TmaArgs {
    const int32_t* tsteps;
    const int64_t* toff;
    const int2* tinfo;
    const int32_t* stream;
    int64_t tpc;
    int W;
    const float* row_scale;
    const float* nbr_scale;
    int self, relu;
    __nv_bfloat16* out;
    float* partial;
};

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// acc[0..7] += the 8 bf16 of v (one mixed-precision add each, as the row-group kernel)
__device__ __forceinline__ void acc8(float (&acc)[8], const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
        unsigned short lo, hi;
        asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w[i]));
        asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc[2 * i]) : "h"(lo));
        asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc[2 * i + 1]) : "h"(hi));
    }
}

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* m, uint32_t bar, int r0, int r1, int r2,
                                        int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}

// consumer-side tile metadata for a window of 32 tiles (lane k holds tile q_base + k): steps,
// and for the warp's two rows the {out, degree} entry and the row / neighbour scales
struct TileWin {
    int32_t ts;
    int2 info0, info1;
    float rs0, rs1, ns0, ns1;
};

__device__ __forceinline__ void load_win(const TmaArgs& a, int64_t qb, int64_t q1, int r0, int lane, TileWin& w) {
    const int64_t q = qb + lane;
    w.ts = 0;
    w.info0 = w.info1 = make_int2(-1, -1);
    w.rs0 = w.rs1 = w.ns0 = w.ns1 = 1.f;
    if (q < q1) {
        w.ts = __ldg(a.tsteps + q);
        const int4 ii = __ldg(reinterpret_cast<const int4*>(a.tinfo + q * kTR + r0));   // rows r0, r0 + 1
        w.info0 = make_int2(ii.x, ii.y);
        w.info1 = make_int2(ii.z, ii.w);
        if (a.row_scale) {
            if (w.info0.x >= 0) w.rs0 = __ldg(a.row_scale + w.info0.x);
            if (w.info1.x >= 0) w.rs1 = __ldg(a.row_scale + w.info1.x);
        }
        if (a.nbr_scale) {
            if (w.info0.x >= 0) w.ns0 = __ldg(a.nbr_scale + w.info0.x);
            if (w.info1.x >= 0) w.ns1 = __ldg(a.nbr_scale + w.info1.x);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 1) k_spmm_tma(const __grid_constant__ CUtensorMap xm, TmaArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing);
    uint64_t* empty = full + kNSlot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q0 = (int64_t)blockIdx.x * a.tpc, q1 = q0 + a.tpc;
    const int64_t s_begin = a.toff[q0], s_end = a.toff[q1];
    const int rowbytes = a.W * 2, stepbytes = kTR * rowbytes;
    const int slot_bytes = kSPC * stepbytes;
    const int R = min(kNSlot, kRing / slot_bytes);          // ring slots (one chunk each)
    if (threadIdx.x == 0) {
        for (int i = 0; i < R; i++) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], kCW);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();
    const int64_t nchunks = ceil_div(s_end - s_begin, kSPC);
    const uint32_t ring_a = tc::smem_u32(ring);
    if (warp >= kCW) {
        // ------------------------------------------------------------- producers
        // warp p fills chunks p, p + kPW, ... ; chunk c lives in ring slot c mod R and may be
        // filled once the consumers released chunk c - R (its slot's previous use)
        const int p = warp - kCW;
        if (p == 0 && lane == 0) tc::tma_prefetch(&xm);
        const int4* quads = reinterpret_cast<const int4*>(a.stream);
        auto load_q = [&](int64_t c) {       // this lane's gather4 row ids of chunk c
            int4 v = make_int4(0, 0, 0, 0);
            if (c < nchunks) {
                const int64_t s0 = s_begin + c * kSPC;
                const int nq = (int)min((int64_t)kSPC, s_end - s0) * (kTR / 4);
                if (lane < nq) v = __ldg(quads + s0 * (kTR / 4) + lane);
            }
            return v;
        };
        int4 qn = load_q(p);
        int slot = p % R;                    // c mod R and c / R, advanced incrementally
        int64_t use = p / R;
        for (int64_t c = p; c < nchunks; c += kPW) {
            const int4 qd = qn;
            qn = load_q(c + kPW);            // the next chunk's row ids, while this one waits
            if (use > 0 && lane == 0) tc::mbar_wait(&empty[slot], (uint32_t)((use - 1) & 1));
            const int64_t s0 = s_begin + c * kSPC;
            const int ns = (int)min((int64_t)kSPC, s_end - s0);
            const int nq = ns * (kTR / 4);
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[slot], (uint32_t)(ns * stepbytes));
            __syncwarp();
            if (lane < nq)
                gather4(ring_a + (uint32_t)(slot * slot_bytes) + (uint32_t)lane * 4u * (uint32_t)rowbytes, &xm,
                        tc::smem_u32(&full[slot]), qd.x, qd.y, qd.z, qd.w);
            slot += kPW;
            while (slot >= R) {
                slot -= R;
                use++;
            }
        }
        return;
    }
    // ----------------------------------------------------------------- consumers
    const int G = a.W >> 3;
    const int half = lane / G, sub = lane - half * G;
    const bool active = half < 2;
    const int r0 = warp * 2;
    const uint32_t lane_off = (uint32_t)((r0 + (active ? half : 0)) * rowbytes + sub * 16);
    // tile metadata: window of 32 tiles, the next window prefetched while this one is used
    TileWin cur, nxt;
    int64_t qb = q0;
    load_win(a, qb, q1, r0, lane, cur);
    load_win(a, qb + 32, q1, r0, lane, nxt);
    int k = 0;                                   // current tile = qb + k
    int32_t j = 0;                               // step within the tile
    int32_t nst = __shfl_sync(0xffffffffu, cur.ts, 0);
    int2 info;
    float rs, ns;
    auto pick = [&]() {
        const int i0x = __shfl_sync(0xffffffffu, cur.info0.x, k), i0y = __shfl_sync(0xffffffffu, cur.info0.y, k);
        const int i1x = __shfl_sync(0xffffffffu, cur.info1.x, k), i1y = __shfl_sync(0xffffffffu, cur.info1.y, k);
        const float a0 = __shfl_sync(0xffffffffu, cur.rs0, k), a1 = __shfl_sync(0xffffffffu, cur.rs1, k);
        const float b0 = __shfl_sync(0xffffffffu, cur.ns0, k), b1 = __shfl_sync(0xffffffffu, cur.ns1, k);
        info = half == 1 ? make_int2(i1x, i1y) : make_int2(i0x, i0y);
        rs = half == 1 ? a1 : a0;
        ns = half == 1 ? b1 : b0;
        nst = __shfl_sync(0xffffffffu, cur.ts, k);
    };
    pick();
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; t++) acc[t] = 0.f;
    uint4 selfv = make_uint4(0, 0, 0, 0);
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t c = 0; c < nchunks; c++) {
        if (c > 0 && ++slot == R) {
            slot = 0;
            phase ^= 1u;
        }
        tc::mbar_wait(&full[slot], phase);
        const int ns_c = (int)min((int64_t)kSPC, s_end - (s_begin + c * kSPC));
        uint32_t src = ring_a + (uint32_t)(slot * slot_bytes) + lane_off;
        if (j >= 1 && j + ns_c < nst) {
            // fast path: the whole chunk lies inside one tile's neighbour steps (j, nst uniform)
            const int valid = active ? min(ns_c, info.y - (j - 1)) : 0;
            if (valid == kSPC) {
                uint4 v[kSPC];
#pragma unroll
                for (int t = 0; t < kSPC; t++) v[t] = lds128(src + (uint32_t)(t * stepbytes));
#pragma unroll
                for (int t = 0; t < kSPC; t++) acc8(acc, v[t]);
            } else {
                for (int t = 0; t < valid; t++) acc8(acc, lds128(src + (uint32_t)(t * stepbytes)));
            }
            j += ns_c;
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[slot]);
            continue;
        }
        for (int s = 0; s < ns_c; s++, src += (uint32_t)stepbytes) {
            if (active) {
                if (j == 0) selfv = lds128(src);
                else if (j - 1 < info.y) acc8(acc, lds128(src));
            }
            if (++j == nst) {
                // the tile's last step: write this row (bf16) or this segment's partial (fp32)
                if (active && info.x != -1) {
                    if ((uint32_t)info.x & kSlotFlag) {
                        float* dst = a.partial + ((int64_t)((uint32_t)info.x & ~kSlotFlag) * G + sub) * 8;
                        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
                        *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
                    } else {
                        const uint32_t w[4] = {selfv.x, selfv.y, selfv.z, selfv.w};
                        uint4 o;
                        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                        for (int t = 0; t < 4; t++) {
                            const float lo = __uint_as_float(w[t] << 16), hi = __uint_as_float(w[t] & 0xffff0000u);
                            float x0 = acc[2 * t], x1 = acc[2 * t + 1];
                            if (a.nbr_scale) { x0 *= ns; x1 *= ns; }
                            if (a.self) { x0 = fmaf(1.f, lo, x0); x1 = fmaf(1.f, hi, x1); }
                            x0 *= rs; x1 *= rs;
                            if (a.relu) { x0 = fmaxf(x0, 0.f); x1 = fmaxf(x1, 0.f); }
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(x0, x1);
                            ow[t] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        *reinterpret_cast<uint4*>(a.out + (int64_t)info.x * a.W + sub * 8) = o;
                    }
                }
#pragma unroll
                for (int t = 0; t < 8; t++) acc[t] = 0.f;
                j = 0;
                if (++k == 32) {                   // next window; prefetch the one after
                    k = 0;
                    qb += 32;
                    cur = nxt;
                    load_win(a, qb + 32, q1, r0, lane, nxt);
                }
                pick();
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[slot]);
    }
}

}  // namespace

bool spmm_tma_eligible(const grappa_ctx* ctx, const SpmmArgs& a, grappa_dtype dt) {
    // bf16 rows of 80..128 elements (two rows per consumer warp), unweighted neighbour sum with a
    // plain self term: every GCN hidden-layer aggregation of the normalised chain (R29)
    return ctx && ctx->var_spmm == 4 && dt == GRAPPA_BF16 && a.width % 16 == 0 && a.width >= 80 &&
           a.width <= 128 && !a.col_scale && !a.edge_w && !a.accumulate && !a.mask && !a.self_sep && !a.X_self &&
           !a.out_compact && a.n > 0 && a.n < (1ll << 31);
}

static grappa_status tma_plan_build(grappa_ctx* ctx, TmaPlan& P, const SpmmArgs& a, cudaStream_t s) {
    const int64_t V = a.n_slots + (a.n - a.n_heavy);
    const int64_t T = ceil_div(V, kTR);
    const int grid = ctx->sm_count;
    const int64_t tpc = std::max<int64_t>(1, ceil_div(T, grid));
    const int64_t nq = (int64_t)grid * tpc;
    // stream size bound without a host sync: rows come in descending degree (<= kSegLen), so
    // sum over row tiles of max degree <= 2 kSegLen + nnz / 16; slot tiles <= kSegLen each
    const int64_t slot_tiles = ceil_div(a.n_slots, kTR) + 1;
    const int64_t steps_bound = nq + (slot_tiles + 2) * kSegLen + a.nnz / kTR + 1;
    GRAPPA_TRY(P.tsteps.grow((size_t)nq * 4));
    GRAPPA_TRY(P.toff.grow((size_t)(nq + 1) * 8));
    GRAPPA_TRY(P.tinfo.grow((size_t)nq * kTR * 8));
    GRAPPA_TRY(P.stream.grow((size_t)steps_bound * kTR * 4));
    PlanSrc p{V, a.n_slots, a.n_heavy, T, a.rowptr, a.slot_row, a.slot_seg, a.row_desc, a.col, grid, tpc};
    const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq, 256), (int64_t)grid * 8));
    k_tma_tile_steps<<<g1, 256, 0, s>>>(p, (int32_t*)P.tsteps.p);
    GRAPPA_LAUNCHED(ctx);
    GRAPPA_TRY(device_scan(ctx, TsRead{(const int32_t*)P.tsteps.p}, nq, TsWrite{(int64_t*)P.toff.p}, s));
    const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq * kTR, 256), (int64_t)grid * 16));
    k_tma_fill<<<g2, 256, 0, s>>>(p, (const int32_t*)P.tsteps.p, (const int64_t*)P.toff.p, (int2*)P.tinfo.p,
                                   (int32_t*)P.stream.p);
    GRAPPA_LAUNCHED(ctx);
    P.grid = grid;
    P.tpc = tpc;
    P.ready = true;
    return GRAPPA_OK;
}

grappa_status spmm_tma(grappa_ctx* ctx, const grappa_part* part, bool transpose, const SpmmArgs& a,
                       cudaStream_t s) {
    TmaPlan& P = transpose ? const_cast<grappa_part*>(part)->t_tma : const_cast<grappa_part*>(part)->tma;
    if (!P.ready) GRAPPA_TRY(tma_plan_build(ctx, P, a, s));
    CUtensorMap xm;
    GRAPPA_TRY(tma_map_rows_bf16(&xm, a.X, a.n, a.width));
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_spmm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    TmaArgs t;
    t.tsteps = (const int32_t*)P.tsteps.p;
    t.toff = (const int64_t*)P.toff.p;
    t.tinfo = (const int2*)P.tinfo.p;
    t.stream = (const int32_t*)P.stream.p;
    t.tpc = P.tpc;
    t.W = a.width;
    t.row_scale = a.row_scale;
    t.nbr_scale = a.nbr_scale;
    t.self = a.self;
    t.relu = a.relu;
    t.out = (__nv_bfloat16*)a.out;
    t.partial = a.partial;
    k_spmm_tma<<<P.grid, kThreads, kSmem, s>>>(xm, t);
    GRAPPA_LAUNCHED(ctx);
    return spmm_fixup(ctx, a, s);
}

}  // namespace grappa
