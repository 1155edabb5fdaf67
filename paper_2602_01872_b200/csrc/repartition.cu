// repartition.cu -- a3: super-epoch repartition = induced chunk-pair subgraph extraction.
//
// PAPER: P:188-198 (§3.3 super-epochs, chunks, partition = base chunk + swept chunk),
// P:413 (§4 "workers load the new chunk's edges"), SPEC S:135-143 (build_partition,
// induced-core mode S:116), S:208 (seeds = core train nodes).
//
// Integer pipeline, bit-exact with the oracle:
//   1. rank table   rank[v] = #core nodes < v (exclusive scan of the core flag), -1 if not
//                   core; core_global[rank[v]] = v  -> local id = ascending global order.
//   2. row count    warp per core row: d_l = popc(ballot(rank[u] >= 0)) over its neighbours,
//                   d_g = global degree; norms, labels, seed flag.
//   3. rowptr       exclusive scan of d_l (int64).  Seeds, split rows, slots: more scans.
//   4. fill         warp per core row: stable ballot compaction of kept neighbours, written
//                   as rank[u] (ascending because the global row is sorted and rank is
//                   monotone).
//   5. features     core rows gathered into local order (16-byte vector copies).
//   6. coverage     fixed-order block partials over the seeds: sum d_l/d_g (f64) and the
//                   exact integers D = sum (d_g - d_l), sum d_l, sum d_g (d_l > 0).
#include <cub/device/device_radix_sort.cuh>

#include "part.cuh"
#include "scan.cuh"

#include <cmath>
#include <cstring>
#include <vector>

namespace grappa {

static size_t al256(size_t b) { return (b + 255) / 256 * 256; }


struct FlagCore {
    const int32_t* chunk_of; int32_t b, s;
    __device__ int32_t operator()(int64_t v) const {
        int32_t c = chunk_of[v];
        return (c == b) | (c == s);
    }
};
struct WriteRank {
    int32_t* rank; int32_t* core_global; int64_t* stat;
    __device__ void operator()(int64_t v, int64_t p, int32_t f) const {
        rank[v] = f ? (int32_t)p : -1;
        if (f) core_global[p] = (int32_t)v;
    }
    __device__ void finish(int64_t, int64_t total) const { stat[0] = total; }
};

struct ReadI32 {
    const int32_t* a;
    __device__ int32_t operator()(int64_t i) const { return a[i]; }
};
struct WriteRowptr {
    int64_t* rowptr; int64_t* stat;
    __device__ void operator()(int64_t i, int64_t p, int32_t) const { rowptr[i] = p; }
    __device__ void finish(int64_t n, int64_t total) const { rowptr[n] = total; stat[1] = total; }
};
struct FlagSeed {
    const int32_t* core_global; const uint8_t* train;
    __device__ int32_t operator()(int64_t i) const { return train[core_global ? core_global[i] : i] != 0; }
};
struct WriteCompact {
    int32_t* out; int64_t* stat; int idx;
    __device__ void operator()(int64_t i, int64_t p, int32_t f) const {
        if (f) out[p] = (int32_t)i;
    }
    __device__ void finish(int64_t, int64_t total) const { stat[idx] = total; }
};
struct FlagHeavy {
    const int32_t* d_l;
    __device__ int32_t operator()(int64_t i) const { return d_l[i] > kSegLen; }
};
struct NumSeg {
    const int32_t* d_l; const int32_t* heavy_rows;
    __device__ int32_t operator()(int64_t h) const {
        return (int32_t)ceil_div(d_l[heavy_rows[h]], kSegLen);
    }
};
struct WriteSlotOff {
    int32_t* slot_off; int64_t* stat; int idx;
    __device__ void operator()(int64_t h, int64_t p, int32_t) const { slot_off[h] = (int32_t)p; }
    __device__ void finish(int64_t n, int64_t total) const { slot_off[n] = (int32_t)total; stat[idx] = total; }
};

// halo-1 (R33): halo = non-core neighbours of core rows; local ids n_core + rank among them
__global__ void k_mark_halo(const int64_t* __restrict__ d_ncore, const int32_t* __restrict__ core_global,
                            const int64_t* __restrict__ g_rowptr, const int32_t* __restrict__ g_col,
                            const int32_t* __restrict__ rank, uint8_t* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t n = *d_ncore;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
        const int32_t v = core_global ? core_global[i] : (int32_t)i;
        for (int64_t e = g_rowptr[v] + lane; e < g_rowptr[v + 1]; e += 32) {
            const int32_t u = g_col[e];
            if (rank[u] < 0) flag[u] = 1;          // idempotent store
        }
    }
}
// the same marking over an explicit CSR with global neighbour ids (a chunk shard: sharded mode)
__global__ void k_mark_halo_rows(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const int32_t* __restrict__ rank, uint8_t* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps)
        for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
            const int32_t u = col[e];
            if (rank[u] < 0) flag[u] = 1;
        }
}
struct FlagHalo {
    const uint8_t* flag;
    __device__ int32_t operator()(int64_t v) const { return flag[v]; }
};
struct WriteHaloRank {
    int32_t* rank; int32_t* core_global; int64_t* stat;
    __device__ void operator()(int64_t v, int64_t p, int32_t f) const {
        if (f) {
            const int64_t id = stat[0] + p;          // after the n_core core nodes
            rank[v] = (int32_t)id;
            core_global[id] = (int32_t)v;
        }
    }
    __device__ void finish(int64_t, int64_t total) const { stat[6] = total; }
};
// halo rows: empty (d_l = 0), GCN norm 1, SAGE norm 0, node weight w = [d_g == 0]
__global__ void k_halo_rows(int64_t n_core, int64_t n_local, const int64_t* __restrict__ d_nnz,
                            const int32_t* __restrict__ core_global, const int64_t* __restrict__ g_rowptr,
                            const int32_t* __restrict__ g_labels, int64_t* rowptr, int32_t* d_l, int32_t* d_g,
                            float* norm_gcn, float* norm_sage, float* node_w, int32_t* labels) {
    const int64_t nnz = *d_nnz;
    for (int64_t i = n_core + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = core_global ? core_global[i] : (int32_t)i;
        // sharded mode: the halo node's global degree and label arrive with its features
        // (grappa_halo_exchange); placeholders until then
        const int32_t dg = g_rowptr ? (int32_t)(g_rowptr[v + 1] - g_rowptr[v]) : 0;
        rowptr[i + 1] = nnz;
        d_l[i] = 0;
        d_g[i] = dg;
        norm_gcn[i] = 1.0f;
        norm_sage[i] = 0.0f;
        const float w = dg == 0 ? 1.0f : 0.0f;
        node_w[i] = w;
        node_w[n_local + i] = w;
        node_w[2 * n_local + i] = 0.0f;
        labels[i] = g_labels ? g_labels[v] : 0;
    }
}
// transpose support: source row of every local edge
__global__ void k_edge_rows(int64_t n_rows, const int64_t* __restrict__ rowptr, int32_t* __restrict__ erow) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nwarps)
        for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) erow[e] = (int32_t)i;
}
// transpose rowptr from the sorted column keys; degree of every transposed row
__global__ void k_t_rowptr(int64_t n, int64_t nnz, const int32_t* __restrict__ skeys, int64_t* __restrict__ trowptr) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cur = e < nnz ? skeys[e] : n;
        const int64_t prev = e > 0 ? skeys[e - 1] : -1;
        for (int64_t r = prev + 1; r <= cur && r <= n; r++) trowptr[r] = e;
    }
}
__global__ void k_iota(int64_t n, int32_t* __restrict__ a) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}
__global__ void k_take(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ src,
                       int32_t* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}
__global__ void k_row_deg(int64_t n, const int64_t* __restrict__ rowptr, int32_t* __restrict__ deg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        deg[i] = (int32_t)(rowptr[i + 1] - rowptr[i]);
}

// Global rows are cut into tasks of at most kTaskLen edges (power-law hubs reach 10^5
// neighbours; a warp takes 32 tasks, so its work is bounded by 32 kTaskLen edges -- the tail
// of a switch is the warp holding a hub's tasks).  Tasks are numbered in
// (row, segment) order, so an exclusive scan of the per-task kept counts is directly each
// task's output offset in the local `col` array -- and the local rowptr.
constexpr int kTaskLen = 128;

struct NumTasks {
    const int32_t* core_global; const int64_t* g_rowptr;
    __device__ int32_t operator()(int64_t i) const {
        const int32_t v = core_global ? core_global[i] : (int32_t)i;
        const int64_t d = g_rowptr[v + 1] - g_rowptr[v];
        return d > kTaskLen ? (int32_t)ceil_div(d, kTaskLen) : 1;
    }
};
// task descriptors {core row, edge count, first edge lo, hi}: the count and fill passes read one
// coalesced 16-byte record per task instead of the dependent row -> core id -> rowptr chain
struct WriteTasks {
    int32_t* task_off; int4* task_desc; int64_t* stat;
    const int32_t* core_global; const int64_t* g_rowptr;
    __device__ void operator()(int64_t i, int64_t p, int32_t k) const {
        task_off[i] = (int32_t)p;
        const int32_t v = core_global ? core_global[i] : (int32_t)i;
        const int64_t e0 = g_rowptr[v], e1 = g_rowptr[v + 1];
        for (int32_t j = 0; j < k; j++) {
            const int64_t a = e0 + (int64_t)j * kTaskLen;
            const int32_t len = (int32_t)min((int64_t)kTaskLen, e1 - a);
            task_desc[p + j] = make_int4((int)i, len, (int)(uint32_t)(a & 0xffffffffll), (int)(a >> 32));
        }
    }
    __device__ void finish(int64_t n, int64_t total) const { task_off[n] = (int32_t)total; stat[5] = total; }
};
struct ReadTcount {
    const int32_t* tcount; const int64_t* d_T;
    __device__ int32_t operator()(int64_t t) const { return t < *d_T ? tcount[t] : 0; }
};
struct WriteTaskOut {
    int64_t* task_out; int64_t* stat;
    __device__ void operator()(int64_t t, int64_t p, int32_t) const { task_out[t] = p; }
    __device__ void finish(int64_t n, int64_t total) const { task_out[n] = total; stat[1] = total; }
};

// kept-neighbour count of every task (warp per task, ballot/popc)
// core membership bitmap of partition {b, s}: bit v = [chunk_of[v] in {b, s}] (warp per 32 nodes)
__global__ void k_core_bitmap(int64_t n, const int32_t* __restrict__ chunk_of, int32_t b, int32_t s,
                              uint32_t* __restrict__ bitmap) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ceil_div(n, 32); w += nw) {
        const int64_t v = w * 32 + lane;
        int32_t c = -1;
        if (v < n) c = chunk_of[v];
        const unsigned m = __ballot_sync(0xffffffffu, c == b || c == s);
        if (lane == 0) bitmap[w] = m;
    }
}
__device__ __forceinline__ bool in_core(const uint32_t* __restrict__ bm, int32_t u) {
    return (__ldg(bm + (u >> 5)) >> (u & 31)) & 1u;
}

// Task processing (count and fill): a warp takes 32 consecutive tasks (one 16-byte descriptor
// per lane, coalesced) and walks them kPackU at a time, all 32 lanes on one task's edges (lane j
// takes edge j, j + 32, ...): the kPackU tasks' col loads and membership probes are independent
// and in flight together, and a task's count is a warp-uniform popc of ballots -- no per-edge
// owner search, no shared-memory bookkeeping.  (Half a warp per task, the former design, left
// most lanes idle on products' short rows and had one dependent descriptor -> col -> bitmap chain
// per task in flight.)  Halo-1 partitions keep every neighbour of a core row (keep_all).
constexpr int kPackU = 4;
// Edge membership in partition {b, s}.  EC: from the per-edge chunk bytes of the global CSR
// (ec[e] = chunk_of[col[e]], built once per (graph, chunk map): a coalesced 1-byte stream
// instead of a dependent random probe per edge); else from the core bitmap (sharded merged CSRs).
struct Member {
    const uint32_t* bitmap;
    const uint8_t* ec;
    int b, s, keep_all;
};
template <bool EC>
__device__ __forceinline__ bool member(const Member& m, int64_t e, int32_t u) {
    if (m.keep_all) return true;
    if (EC) {
        const int c = __ldg(m.ec + e);
        return c == m.b || c == m.s;
    }
    return in_core(m.bitmap, u);
}
template <bool EC>
__global__ void __launch_bounds__(256, 6) k_task_count(const int64_t* __restrict__ d_T,
                                                    const int4* __restrict__ task_desc,
                                                    const int32_t* __restrict__ g_col, Member mb,
                                                    int32_t* __restrict__ tcount) {
    const int lane = threadIdx.x & 31;
    const int64_t T = *d_T;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; t0 < T; t0 += nwarps * 32) {
        int32_t len = 0;
        int64_t e0 = 0;
        if (t0 + lane < T) {
            const int4 d = __ldg(task_desc + t0 + lane);
            len = d.y;
            e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
        }
        if (mb.keep_all) {
            if (t0 + lane < T) tcount[t0 + lane] = len;
            continue;
        }
        const int nt = (int)min((int64_t)32, T - t0);
        int32_t mine = 0;                       // lane i ends with task i's count
        for (int i = 0; i < nt; i += kPackU) {
            int32_t L[kPackU], c[kPackU];
            int64_t E[kPackU];
#pragma unroll
            for (int k = 0; k < kPackU; k++) {
                L[k] = __shfl_sync(0xffffffffu, len, (i + k) & 31);
                E[k] = __shfl_sync(0xffffffffu, e0, (i + k) & 31);
                if (i + k >= nt) L[k] = 0;
                c[k] = 0;
            }
            int32_t Lm = L[0];
#pragma unroll
            for (int k = 1; k < kPackU; k++) Lm = max(Lm, L[k]);
            for (int32_t off = 0; off < Lm; off += 32) {
                bool kp[kPackU];
                if (EC) {        // only the chunk bytes are needed to count
#pragma unroll
                    for (int k = 0; k < kPackU; k++) kp[k] = off + lane < L[k] && member<true>(mb, E[k] + off + lane, 0);
                } else {
                    int32_t u[kPackU];
#pragma unroll
                    for (int k = 0; k < kPackU; k++) u[k] = off + lane < L[k] ? __ldg(g_col + E[k] + off + lane) : -1;
#pragma unroll
                    for (int k = 0; k < kPackU; k++) kp[k] = u[k] >= 0 && member<false>(mb, 0, u[k]);
                }
#pragma unroll
                for (int k = 0; k < kPackU; k++) c[k] += __popc(__ballot_sync(0xffffffffu, kp[k]));
            }
#pragma unroll
            for (int k = 0; k < kPackU; k++)
                if (lane == i + k) mine = c[k];
        }
        if (t0 + lane < T) tcount[t0 + lane] = mine;
    }
}

// per core row: local rowptr / d_l from the task offsets, d_g, norms, labels
__global__ void k_row_finalize(int64_t n_core, const int32_t* __restrict__ task_off,
                               const int64_t* __restrict__ task_out, const int32_t* __restrict__ core_global,
                               const int64_t* __restrict__ g_rowptr, const int32_t* __restrict__ g_labels,
                               int64_t* rowptr, int32_t* d_l, int32_t* d_g, float* norm_gcn, float* norm_sage,
                               float* node_w, int64_t w_stride, int32_t* labels,
                               unsigned long long* __restrict__ sum_dg) {
    unsigned long long my_dg = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_core;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = task_out[task_off[i]], b = task_out[task_off[i + 1]];
        const int32_t v = core_global ? core_global[i] : (int32_t)i;
        const int32_t cnt = (int32_t)(b - a);
        rowptr[i] = a;
        if (i == n_core - 1) rowptr[n_core] = b;
        d_l[i] = cnt;
        const int32_t dg = (int32_t)(g_rowptr[v + 1] - g_rowptr[v]);
        d_g[i] = dg;
        my_dg += (unsigned long long)dg;
        const double ng = 1.0 / sqrt((double)cnt + 1.0), ns = cnt > 0 ? 1.0 / (double)cnt : 0.0;
        norm_gcn[i] = (float)ng;
        norm_sage[i] = (float)ns;
        // node-level estimator (eq. (9), R30): w = d_l/d_g, 1 iff d_g = 0
        const double w = dg == 0 ? 1.0 : (double)cnt / (double)dg;
        node_w[i] = (float)w;
        node_w[w_stride + i] = (float)(w * ng);
        node_w[2 * w_stride + i] = (float)(w * ns);
        labels[i] = g_labels ? g_labels[v] : 0;
    }
    // sum of the core rows' global degrees (integer, order-free): the rows' source bytes for the
    // algorithmic byte count of the profiling scope
    my_dg = warp_sum(my_dg);
    if ((threadIdx.x & 31) == 0 && my_dg) atomicAdd(sum_dg, my_dg);
}

// stable compaction of every task's kept neighbours (walked like k_task_count): a kept edge goes
// to its task's offset + the task's kept edges before it (a warp-uniform running count + the popc
// of the lower lanes).  It writes the GLOBAL neighbour id; k_relabel then maps every entry through
// the rank table in one fully parallel pass -- the dependent rank probe per kept edge inside the
// walk (col -> membership -> rank -> store) was what bounded the fill.
template <bool EC>
__global__ void __launch_bounds__(256, 6) k_task_fill(const int64_t* __restrict__ d_T,
                                                   const int4* __restrict__ task_desc,
                                                   const int64_t* __restrict__ task_out,
                                                   const int32_t* __restrict__ g_col, Member mb,
                                                   int32_t* __restrict__ col) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t T = *d_T;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; t0 < T; t0 += nwarps * 32) {
        int32_t len = 0;
        int64_t e0 = 0, out = 0;
        if (t0 + lane < T) {
            const int4 d = __ldg(task_desc + t0 + lane);
            len = d.y;
            e0 = (int64_t)(uint32_t)d.z | ((int64_t)d.w << 32);
            out = task_out[t0 + lane];
        }
        const int nt = (int)min((int64_t)32, T - t0);
        for (int i = 0; i < nt; i += kPackU) {
            int32_t L[kPackU];
            int64_t E[kPackU], O[kPackU];
#pragma unroll
            for (int k = 0; k < kPackU; k++) {
                L[k] = __shfl_sync(0xffffffffu, len, (i + k) & 31);
                E[k] = __shfl_sync(0xffffffffu, e0, (i + k) & 31);
                O[k] = __shfl_sync(0xffffffffu, out, (i + k) & 31);
                if (i + k >= nt) L[k] = 0;
            }
            int32_t Lm = L[0];
#pragma unroll
            for (int k = 1; k < kPackU; k++) Lm = max(Lm, L[k]);
            for (int32_t off = 0; off < Lm; off += 32) {
                int32_t u[kPackU];
                bool keep[kPackU];
                if (EC) {
                    // the chunk byte and the neighbour id are independent loads: issue all 2 x kPackU
                    // together (a membership test behind the id load serialised the two latencies)
                    bool in[kPackU];
                    int c[kPackU];
#pragma unroll
                    for (int k = 0; k < kPackU; k++) in[k] = off + lane < L[k];
#pragma unroll
                    for (int k = 0; k < kPackU; k++) {
                        u[k] = in[k] ? __ldg(g_col + E[k] + off + lane) : -1;
                        c[k] = in[k] ? (int)__ldg(mb.ec + E[k] + off + lane) : -1;
                    }
#pragma unroll
                    for (int k = 0; k < kPackU; k++)
                        keep[k] = in[k] && (mb.keep_all || c[k] == mb.b || c[k] == mb.s);
                } else {
#pragma unroll
                    for (int k = 0; k < kPackU; k++) u[k] = off + lane < L[k] ? __ldg(g_col + E[k] + off + lane) : -1;
#pragma unroll
                    for (int k = 0; k < kPackU; k++) keep[k] = u[k] >= 0 && member<EC>(mb, E[k] + off + lane, u[k]);
                }
#pragma unroll
                for (int k = 0; k < kPackU; k++) {
                    const unsigned bal = __ballot_sync(0xffffffffu, keep[k]);
                    if (keep[k]) col[O[k] + __popc(bal & below)] = u[k];
                    O[k] += __popc(bal);
                }
            }
        }
    }
}

// global -> local neighbour ids of a partition's CSR through its rank table (independent loads)
__global__ void k_relabel(int64_t nnz, const int32_t* __restrict__ rank, int32_t* __restrict__ col) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        col[e] = __ldg(rank + col[e]);
}

__global__ void k_slot_tasks(int64_t n_heavy, const int32_t* heavy_rows, const int32_t* slot_off,
                             int32_t* slot_row, int32_t* slot_seg) {
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < n_heavy;
         h += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = heavy_rows[h];
        for (int32_t t = slot_off[h], sgi = 0; t < slot_off[h + 1]; t++, sgi++) {
            slot_row[t] = r;
            slot_seg[t] = sgi;
        }
    }
}

__global__ void k_gather_rows(int64_t n_core, int64_t row_bytes, const int32_t* __restrict__ core_global,
                              const uint4* __restrict__ src, uint4* __restrict__ dst) {
    // one thread per 16-byte vector of the output (every lane busy whatever the row width)
    const int64_t vec = row_bytes / 16;
    const int64_t total = n_core * vec;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / vec, k = i - r * vec;
        dst[i] = __ldg(src + (int64_t)__ldg(core_global + r) * vec + k);
    }
}

// Degree-bucketed SpMM row order (bucket 0 = heaviest); order inside a bucket is arbitrary
// (it only decides which warp processes a row, never a result).
constexpr int kDegBuckets = kSegLen + 2;
__device__ __forceinline__ int deg_bucket(int32_t d) { return kSegLen + 1 - min(d, kSegLen + 1); }

__global__ void k_deg_hist(int64_t n, const int32_t* __restrict__ d_l, unsigned long long* bins) {
    __shared__ unsigned int sh[kDegBuckets];
    for (int i = threadIdx.x; i < kDegBuckets; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&sh[deg_bucket(d_l[i])], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kDegBuckets; i += blockDim.x)
        if (sh[i]) atomicAdd(&bins[i], (unsigned long long)sh[i]);
}

// exclusive scan of the bucket counts by one warp (each lane a contiguous run of buckets)
__global__ void k_deg_bins_scan(const unsigned long long* bins, unsigned long long* cursor) {
    constexpr int kPer = (kDegBuckets + 31) / 32;
    const int lane = threadIdx.x & 31;
    unsigned long long v[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int i = lane * kPer + k;
        v[k] = i < kDegBuckets ? bins[i] : 0ull;
        sum += v[k];
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    unsigned long long run = incl - sum;
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int i = lane * kPer + k;
        if (i < kDegBuckets) cursor[i] = run;
        run += v[k];
    }
}

// each block owns a contiguous run of rows: counts its buckets in shared memory, reserves one
// range per bucket with a single global atomic, then places its rows (no hot global counter)
__global__ void k_deg_scatter(int64_t n, int64_t per_block, const int32_t* __restrict__ d_l,
                              unsigned long long* cursor, int32_t* __restrict__ order) {
    __shared__ unsigned int cnt[kDegBuckets];
    __shared__ unsigned long long base[kDegBuckets];
    const int64_t r0 = (int64_t)blockIdx.x * per_block, r1 = min(n, r0 + per_block);
    for (int i = threadIdx.x; i < kDegBuckets; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicAdd(&cnt[deg_bucket(d_l[i])], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kDegBuckets; i += blockDim.x) {
        base[i] = cnt[i] ? atomicAdd(&cursor[i], (unsigned long long)cnt[i]) : 0ull;
        cnt[i] = 0;
    }
    __syncthreads();
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const int b = deg_bucket(d_l[i]);
        order[base[b] + atomicAdd(&cnt[b], 1u)] = (int32_t)i;
    }
}

__global__ void k_row_desc(int64_t n, const int32_t* __restrict__ order, const int64_t* __restrict__ rowptr,
                           int4* __restrict__ desc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = order[i];
        const int64_t e0 = rowptr[v];
        desc[i] = make_int4(v, (int)(rowptr[v + 1] - e0), (int)(uint32_t)(e0 & 0xffffffffll), (int)(e0 >> 32));
    }
}

// Coverage statistics over the seeds, fixed-order block partials.
struct SeedStats {
    double sum_r;      // sum d_l/d_g (ratio 1 where d_g = 0), R4
    long long D;       // sum_{d_l>0} (d_g - d_l)
    long long sum_dl;  // sum_{d_l>0} d_l
    long long sum_dg;  // sum_{d_l>0} d_g
};

constexpr int kStatThreads = 256;

__device__ SeedStats block_reduce_stats(SeedStats v) {
    __shared__ SeedStats sh[kStatThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v.sum_r = warp_sum(v.sum_r);
    v.D = warp_sum(v.D);
    v.sum_dl = warp_sum(v.sum_dl);
    v.sum_dg = warp_sum(v.sum_dg);
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    SeedStats t{0, 0, 0, 0};
    if (threadIdx.x == 0)
        for (int w = 0; w < kStatThreads / 32; w++) {
            t.sum_r += sh[w].sum_r; t.D += sh[w].D; t.sum_dl += sh[w].sum_dl; t.sum_dg += sh[w].sum_dg;
        }
    return t;
}

__global__ void k_seed_stats(int64_t n_seeds, const int32_t* seeds, const int32_t* d_l,
                             const int32_t* d_g, SeedStats* part) {
    SeedStats a{0, 0, 0, 0};
    const int64_t per = ceil_div(n_seeds, gridDim.x);
    const int64_t s0 = blockIdx.x * per, s1 = min(n_seeds, s0 + per);
    for (int64_t k = s0 + threadIdx.x; k < s1; k += blockDim.x) {
        const int32_t i = seeds[k];
        const int32_t l = d_l[i], g = d_g[i];
        a.sum_r += g == 0 ? 1.0 : (double)l / (double)g;
        if (l > 0) { a.D += g - l; a.sum_dl += l; a.sum_dg += g; }
    }
    SeedStats t = block_reduce_stats(a);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_seed_stats_final(int nb, const SeedStats* part, SeedStats* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        SeedStats t{0, 0, 0, 0};
        for (int b = 0; b < nb; b++) {
            t.sum_r += part[b].sum_r; t.D += part[b].D; t.sum_dl += part[b].sum_dl; t.sum_dg += part[b].sum_dg;
        }
        *out = t;
    }
}

}  // namespace grappa

using namespace grappa;

// blocks of the fixed-order coverage-statistics reduction (the same for every path, so the f64
// sums are identical whichever call built the partition)
static int seed_stat_blocks(const grappa_ctx* ctx, int64_t n_seeds) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_seeds, 512), (int64_t)ctx->sm_count * 4));
}

static grappa_status rp_grid(grappa_ctx* ctx, int64_t rows, int threads, unsigned* grid) {
    int64_t warps_per_block = threads / 32;
    int64_t b = ceil_div(rows, warps_per_block);
    int64_t cap = (int64_t)ctx->sm_count * 16;
    *grid = (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
    return GRAPPA_OK;
}

// SpMM plan of one CSR: rows with deg > kSegLen split into kSegLen-edge slots (fixed-order
// fix-up combine), degree-bucketed row order, 16-byte row descriptors.  Two host syncs (the
// split-row and slot counts size the slot tables).
struct PlanBufs {
    DevBuf *heavy_rows, *heavy_slot_off, *slot_row, *slot_seg, *row_order, *row_desc;
};
static grappa_status plan_order(grappa_ctx* ctx, cudaStream_t s, int64_t n, const int64_t* rowptr,
                                const int32_t* deg, PlanBufs b, unsigned long long* bins = nullptr);
static grappa_status build_plan(grappa_ctx* ctx, cudaStream_t s, int64_t n, const int64_t* rowptr,
                                const int32_t* deg, PlanBufs b, int64_t* d_st, int64_t* n_heavy_out,
                                int64_t* n_slots_out) {
    GRAPPA_TRY(b.heavy_rows->grow((size_t)(n > 0 ? n : 1) * 4));
    GRAPPA_TRY(b.heavy_slot_off->grow((size_t)(n + 1) * 4));
    GRAPPA_TRY(device_scan(ctx, FlagHeavy{deg}, n, WriteCompact{(int32_t*)b.heavy_rows->p, d_st, 0}, s));
    int64_t n_heavy = 0;
    GRAPPA_CUDA(cudaMemcpyAsync(&n_heavy, d_st, 8, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    int64_t n_slots = 0;
    if (n_heavy > 0) {
        GRAPPA_TRY(device_scan(ctx, NumSeg{deg, (int32_t*)b.heavy_rows->p}, n_heavy,
                               WriteSlotOff{(int32_t*)b.heavy_slot_off->p, d_st, 1}, s));
        GRAPPA_CUDA(cudaMemcpyAsync(&n_slots, d_st + 1, 8, cudaMemcpyDeviceToHost, s));
        GRAPPA_CUDA(cudaStreamSynchronize(s));
    }
    GRAPPA_TRY(b.slot_row->grow((size_t)(n_slots > 0 ? n_slots : 1) * 4));
    GRAPPA_TRY(b.slot_seg->grow((size_t)(n_slots > 0 ? n_slots : 1) * 4));
    if (n_heavy > 0) {
        k_slot_tasks<<<(unsigned)std::min<int64_t>(ceil_div(n_heavy, 256), 1024), 256, 0, s>>>(
            n_heavy, (int32_t*)b.heavy_rows->p, (int32_t*)b.heavy_slot_off->p, (int32_t*)b.slot_row->p,
            (int32_t*)b.slot_seg->p);
        GRAPPA_LAUNCHED(ctx);
    }
    // row order: counting sort by descending min(deg, kSegLen + 1)
    GRAPPA_TRY(b.row_order->grow((size_t)(n > 0 ? n : 1) * 4));
    GRAPPA_TRY(ctx->red_ws.grow((size_t)2 * kDegBuckets * 8));
    *n_heavy_out = n_heavy;
    *n_slots_out = n_slots;
    return plan_order(ctx, s, n, rowptr, deg, b);
}

// degree-bucketed row order (counting sort) and the 16-byte row descriptors of a local CSR
static grappa_status plan_order(grappa_ctx* ctx, cudaStream_t s, int64_t n, const int64_t* rowptr,
                                const int32_t* deg, PlanBufs b, unsigned long long* bins) {
    if (!bins) bins = (unsigned long long*)ctx->red_ws.p;
    GRAPPA_CUDA(cudaMemsetAsync(bins, 0, (size_t)kDegBuckets * 8, s));
    const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 8));
    k_deg_hist<<<g2, 256, 0, s>>>(n, deg, bins);
    GRAPPA_LAUNCHED(ctx);
    k_deg_bins_scan<<<1, 32, 0, s>>>(bins, bins + kDegBuckets);
    GRAPPA_LAUNCHED(ctx);
    const int64_t per = 4096;
    if (n > 0) {
        k_deg_scatter<<<(unsigned)ceil_div(n, per), 256, 0, s>>>(n, per, deg, bins + kDegBuckets,
                                                                 (int32_t*)b.row_order->p);
        GRAPPA_LAUNCHED(ctx);
    }
    GRAPPA_TRY(b.row_desc->grow((size_t)(n > 0 ? n : 1) * 16));
    k_row_desc<<<g2, 256, 0, s>>>(n, (int32_t*)b.row_order->p, rowptr, (int4*)b.row_desc->p);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

// build_plan with the split-row sizes known (batched switch): no host sync
// (ws / bins: a side stream's own scan partials and bucket counters; null = the ctx's)
static grappa_status build_plan_sized(grappa_ctx* ctx, cudaStream_t s, int64_t n, const int64_t* rowptr,
                                      const int32_t* deg, PlanBufs b, int64_t* d_st, int64_t n_heavy,
                                      int64_t n_slots, DevBuf* ws = nullptr, unsigned long long* bins = nullptr) {
    GRAPPA_TRY(b.heavy_rows->grow((size_t)(n > 0 ? n : 1) * 4));
    GRAPPA_TRY(b.heavy_slot_off->grow((size_t)(n_heavy + 1) * 4));
    GRAPPA_TRY(b.slot_row->grow((size_t)(n_slots > 0 ? n_slots : 1) * 4));
    GRAPPA_TRY(b.slot_seg->grow((size_t)(n_slots > 0 ? n_slots : 1) * 4));
    if (n_heavy > 0) {
        GRAPPA_TRY(device_scan(ctx, FlagHeavy{deg}, n, WriteCompact{(int32_t*)b.heavy_rows->p, d_st, 0}, s,
                               nullptr, ws));
        GRAPPA_TRY(device_scan(ctx, NumSeg{deg, (int32_t*)b.heavy_rows->p}, n_heavy,
                               WriteSlotOff{(int32_t*)b.heavy_slot_off->p, d_st, 1}, s, nullptr, ws));
        k_slot_tasks<<<(unsigned)std::min<int64_t>(ceil_div(n_heavy, 256), 1024), 256, 0, s>>>(
            n_heavy, (int32_t*)b.heavy_rows->p, (int32_t*)b.heavy_slot_off->p, (int32_t*)b.slot_row->p,
            (int32_t*)b.slot_seg->p);
        GRAPPA_LAUNCHED(ctx);
    }
    GRAPPA_TRY(b.row_order->grow((size_t)(n > 0 ? n : 1) * 4));
    if (!bins) GRAPPA_TRY(ctx->red_ws.grow((size_t)2 * kDegBuckets * 8));
    return plan_order(ctx, s, n, rowptr, deg, b, bins);
}

extern "C" grappa_status grappa_repartition(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                            int32_t feat_dim, grappa_dtype dtype,
                                            const int32_t* chunk_of, int32_t num_chunks,
                                            int32_t base, int32_t swept, const uint8_t* train_mask,
                                            const int32_t* labels, grappa_part** inout,
                                            void* stream) {
    CallScope call_scope(ctx, stream);
    return grappa_repartition_ex(ctx, g, feats, feat_dim, dtype, chunk_of, num_chunks, base, swept,
                                 train_mask, labels, 0u, inout, stream);
}

static grappa_status repart_impl(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                 int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                 int32_t num_chunks, int32_t base, int32_t swept, const uint8_t* train_mask,
                                 const int32_t* labels, unsigned flags, const grappa_shard* sa,
                                 const grappa_shard* sb, grappa_part** inout, cudaStream_t s) {
    GRAPPA_ARG((flags & ~GRAPPA_PART_HALO1) == 0, GRAPPA_E_ARG, "grappa_repartition_ex: flags 0x%x invalid",
               flags);
    GRAPPA_ARG(base != swept, GRAPPA_E_ARG, "grappa_repartition: base == swept (S:139)");
    GRAPPA_ARG(base >= 0 && swept >= 0 && base < num_chunks && swept < num_chunks, GRAPPA_E_ARG,
               "grappa_repartition: chunk id out of range");
    GRAPPA_ARG(feats == nullptr || (feat_dim > 0 && feat_dim % 16 == 0), GRAPPA_E_SHAPE,
               "grappa_repartition: feat_dim must be a positive multiple of 16");
    GRAPPA_ARG(g->num_nodes > 0 && g->num_nodes < (1ll << 31), GRAPPA_E_ARG,
               "grappa_repartition: num_nodes out of int32 range");
    const bool halo = flags & GRAPPA_PART_HALO1;
    ProfScope ps(ctx, s, GRAPPA_K_REPART, 0.0, 0.0);
    grappa_part* p = *inout ? *inout : new grappa_part();
    const int64_t N = g->num_nodes;
    auto fail = [&](grappa_status st) {
        if (!*inout) {
            grappa_part_destroy(p);
        }
        return st;
    };
#define RP_TRY(expr)                               \
    do {                                           \
        grappa_status _s = (expr);                 \
        if (_s != GRAPPA_OK) return fail(_s);      \
    } while (0)

    // stats: [0]=n_core [1]=nnz [2]=n_seeds [3]=n_heavy [4]=n_slots [5]=T [6]=n_halo ; then SeedStats
    RP_TRY(ctx->small.grow(16 * sizeof(int64_t) + sizeof(SeedStats)));
    int64_t* d_stat = (int64_t*)ctx->small.p;
    SeedStats* d_seedstats = (SeedStats*)(d_stat + 8);
    // rank table (int32 [N]) + halo flags (uint8 [N], halo-1 only)
    const int64_t n_words = ceil_div(N, 32);
    RP_TRY(ctx->red_ws.grow((size_t)N * sizeof(int32_t) + (size_t)n_words * 4 + (halo ? (size_t)N : 0)));
    int32_t* rank = (int32_t*)ctx->red_ws.p;
    uint32_t* bitmap = (uint32_t*)(rank + N);          // core membership (the per-edge test)
    uint8_t* hflag = (uint8_t*)(bitmap + n_words);
    // 1. rank table.  core_global capacity: N (freed/reused across super-epochs)
    RP_TRY(p->core_global.grow((size_t)N * sizeof(int32_t)));
    RP_TRY(device_scan(ctx, FlagCore{chunk_of, base, swept}, N,
                       WriteRank{rank, (int32_t*)p->core_global.p, d_stat}, s));
    if (halo) {
        // 1b. halo = non-core neighbours of core rows; they extend the rank table after the core
        GRAPPA_CUDA(cudaMemsetAsync(hflag, 0, (size_t)N, s));
        if (sa) {        // the two shards' rows carry the core rows' global adjacency
            for (const grappa_shard* sh : {sa, sb}) {
                k_mark_halo_rows<<<(unsigned)ctx->sm_count * 16, 256, 0, s>>>(sh->info.n_rows, sh->info.rowptr,
                                                                               sh->info.col, rank, hflag);
                GRAPPA_LAUNCHED(ctx);
            }
        } else {
            k_mark_halo<<<(unsigned)ctx->sm_count * 16, 256, 0, s>>>(d_stat, (int32_t*)p->core_global.p,
                                                                      g->rowptr, g->col, rank, hflag);
            GRAPPA_LAUNCHED(ctx);
        }
        RP_TRY(device_scan(ctx, FlagHalo{hflag}, N, WriteHaloRank{rank, (int32_t*)p->core_global.p, d_stat}, s));
    } else {
        GRAPPA_CUDA(cudaMemsetAsync(d_stat + 6, 0, 8, s));
    }
    int64_t cnt2[7];
    if (cudaMemcpyAsync(cnt2, d_stat, 7 * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("grappa_repartition: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    const int64_t n_core = cnt2[0], n_halo = cnt2[6], n_local = n_core + n_halo;
    GRAPPA_ARG(n_core > 0, fail(GRAPPA_E_EMPTY), "grappa_repartition: empty partition");
    // Source rows.  Replicated: row v of the global CSR for core row i (v = core_global[i]);
    // sharded: the two shards merged into one CSR in local order (row i = core row i).
    const int32_t* srow = (const int32_t*)p->core_global.p;
    const int64_t* G_rowptr = g->rowptr;
    const int32_t* G_col = g->col;
    int64_t G_nnz = g->nnz;
    const int32_t* G_labels = labels;
    const uint8_t* G_train = train_mask;
    const int64_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
    if (sa) {
        G_nnz = sa->info.nnz + sb->info.nnz;
        const size_t a_src = al256((size_t)n_core * 8), a_deg = al256((size_t)n_core * 4),
                     a_rp = al256((size_t)(n_core + 1) * 8), a_col = al256((size_t)(G_nnz > 0 ? G_nnz : 1) * 4),
                     a_lab = al256((size_t)n_core * 4), a_tr = al256((size_t)n_core);
        RP_TRY(ctx->sh_ws.grow(a_src + a_deg + a_rp + a_col + a_lab + a_tr));
        char* w = (char*)ctx->sh_ws.p;
        int64_t* m_src = (int64_t*)w; w += a_src;
        int32_t* m_deg = (int32_t*)w; w += a_deg;
        int64_t* m_rowptr = (int64_t*)w; w += a_rp;
        int32_t* m_col = (int32_t*)w; w += a_col;
        int32_t* m_lab = (int32_t*)w; w += a_lab;
        uint8_t* m_tr = (uint8_t*)w;
        if (feats) RP_TRY(p->x.grow((size_t)n_local * feat_dim * esz));   // halo rows: grappa_halo_exchange
        RP_TRY(shard_merge(ctx, sa, sb, rank, n_core, m_src, m_deg, m_rowptr, m_col, m_lab, m_tr,
                           feats ? p->x.p : nullptr, feat_dim * esz, d_stat, s));
        srow = nullptr;
        G_rowptr = m_rowptr; G_col = m_col; G_labels = m_lab; G_train = m_tr;
    }
    // 2. per-row counts (core rows from their global rows; halo rows are empty)
    RP_TRY(p->d_l.grow(n_local * 4));
    RP_TRY(p->d_g.grow(n_local * 4));
    RP_TRY(p->norm_gcn.grow(n_local * 4));
    RP_TRY(p->norm_sage.grow(n_local * 4));
    RP_TRY(p->node_w.grow(n_local * 12));
    RP_TRY(p->labels.grow(n_local * 4));
    RP_TRY(p->rowptr.grow((n_local + 1) * 8));
    RP_TRY(p->seeds.grow(n_core * 4));
    unsigned grid;
    rp_grid(ctx, n_local, 256, &grid);
    // task workspace: T <= n_core + nnz_global / kTaskLen + 1 (upper bound; the exact T stays
    // on the device and the task kernels grid-stride up to it -- no host sync needed)
    const int64_t T_max = n_core + G_nnz / kTaskLen + 1;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t off_b = al((size_t)(n_core + 1) * 4), row_b = al((size_t)T_max * 16),
                 cnt_b = al((size_t)T_max * 4), out_b = al((size_t)(T_max + 1) * 8);
    RP_TRY(ctx->rp_ws.grow(off_b + row_b + cnt_b + out_b));
    int32_t* task_off = (int32_t*)ctx->rp_ws.p;
    int4* task_desc = (int4*)((char*)ctx->rp_ws.p + off_b);
    int32_t* tcount = (int32_t*)((char*)ctx->rp_ws.p + off_b + row_b);
    int64_t* task_out = (int64_t*)((char*)ctx->rp_ws.p + off_b + row_b + cnt_b);
    const int32_t* core_global = (const int32_t*)p->core_global.p;
    RP_TRY(device_scan(ctx, NumTasks{srow, G_rowptr}, n_core,
                       WriteTasks{task_off, task_desc, d_stat, srow, G_rowptr}, s));
    const unsigned tgrid = (unsigned)ctx->sm_count * 16;
    // membership: the core bitmap; halo-1 keeps every neighbour
    const uint8_t* ec = nullptr;         // (the per-edge chunk bytes live in a grappa_index)
    if (!halo) {
        k_core_bitmap<<<(unsigned)ctx->sm_count * 16, 256, 0, s>>>(N, chunk_of, base, swept, bitmap);
        GRAPPA_LAUNCHED(ctx);
    }
    const Member mb{bitmap, ec, base, swept, halo ? 1 : 0};
    if (ec) k_task_count<true><<<tgrid, 256, 0, s>>>(d_stat + 5, task_desc, G_col, mb, tcount);
    else k_task_count<false><<<tgrid, 256, 0, s>>>(d_stat + 5, task_desc, G_col, mb, tcount);
    GRAPPA_LAUNCHED(ctx);
    // 3. scans: task outputs (= local col offsets, total = nnz), then per-row finalize
    RP_TRY(device_scan(ctx, ReadTcount{tcount, d_stat + 5}, T_max, WriteTaskOut{task_out, d_stat}, s));
    GRAPPA_CUDA(cudaMemsetAsync(d_stat + 7, 0, 8, s));      // sum of d_g (k_row_finalize)
    k_row_finalize<<<grid, 256, 0, s>>>(n_core, task_off, task_out, srow, G_rowptr, G_labels,
                                         (int64_t*)p->rowptr.p, (int32_t*)p->d_l.p, (int32_t*)p->d_g.p,
                                         (float*)p->norm_gcn.p, (float*)p->norm_sage.p,
                                         (float*)p->node_w.p, n_local, (int32_t*)p->labels.p,
                                         (unsigned long long*)(d_stat + 7));
    GRAPPA_LAUNCHED(ctx);
    if (halo && n_halo > 0) {
        // (sharded: the labels argument is the base shard's, indexed by shard row -- the halo rows'
        // labels and degrees come with grappa_halo_exchange)
        k_halo_rows<<<grid, 256, 0, s>>>(n_core, n_local, d_stat + 1, core_global, sa ? nullptr : g->rowptr,
                                          sa ? nullptr : labels,
                                          (int64_t*)p->rowptr.p, (int32_t*)p->d_l.p, (int32_t*)p->d_g.p,
                                          (float*)p->norm_gcn.p, (float*)p->norm_sage.p,
                                          (float*)p->node_w.p, (int32_t*)p->labels.p);
        GRAPPA_LAUNCHED(ctx);
    }
    RP_TRY(device_scan(ctx, FlagSeed{srow, G_train}, n_core,
                       WriteCompact{(int32_t*)p->seeds.p, d_stat, 2}, s));
    int64_t st[3];
    if (cudaMemcpyAsync(st, d_stat, 3 * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("grappa_repartition: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    const int64_t nnz = st[1], n_seeds = st[2];
    GRAPPA_ARG(n_seeds > 0, fail(GRAPPA_E_EMPTY),
               "grappa_repartition: partition (%d,%d) has no seeds (S:213)", base, swept);
    // 4. fill
    RP_TRY(p->col.grow((size_t)(nnz > 0 ? nnz : 1) * 4));
    if (ec) k_task_fill<true><<<tgrid, 256, 0, s>>>(d_stat + 5, task_desc, task_out, G_col, mb, (int32_t*)p->col.p);
    else k_task_fill<false><<<tgrid, 256, 0, s>>>(d_stat + 5, task_desc, task_out, G_col, mb, (int32_t*)p->col.p);
    GRAPPA_LAUNCHED(ctx);
    if (nnz > 0) {
        k_relabel<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), (int64_t)ctx->sm_count * 32), 256, 0, s>>>(
            nnz, rank, (int32_t*)p->col.p);
    }
    GRAPPA_LAUNCHED(ctx);
    // 5. features (core and halo rows)
    if (feats && !sa) {
        RP_TRY(p->x.grow((size_t)n_local * feat_dim * esz));
        k_gather_rows<<<grid, 256, 0, s>>>(n_local, feat_dim * esz, (int32_t*)p->core_global.p,
                                           (const uint4*)feats, (uint4*)p->x.p);
        GRAPPA_LAUNCHED(ctx);
    }
    // 6. coverage statistics over the seeds (R3; in halo-1 mode every seed has d_l = d_g, R33)
    int nb = seed_stat_blocks(ctx, n_seeds);
    if (nb < 1) nb = 1;
    RP_TRY(ctx->scan_ws.grow((size_t)nb * sizeof(SeedStats)));
    k_seed_stats<<<nb, kStatThreads, 0, s>>>(n_seeds, (int32_t*)p->seeds.p, (int32_t*)p->d_l.p,
                                              (int32_t*)p->d_g.p, (SeedStats*)ctx->scan_ws.p);
    GRAPPA_LAUNCHED(ctx);
    k_seed_stats_final<<<1, 32, 0, s>>>(nb, (SeedStats*)ctx->scan_ws.p, d_seedstats);
    GRAPPA_LAUNCHED(ctx);
    SeedStats hs;
    int64_t sum_dg = 0;
    if (cudaMemcpyAsync(&hs, d_seedstats, sizeof(hs), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&sum_dg, d_stat + 7, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        set_error("grappa_repartition: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    // 7. SpMM plan of the local CSR (split rows, row order, descriptors)
    int64_t n_heavy = 0, n_slots = 0;
    RP_TRY(build_plan(ctx, s, n_local, (int64_t*)p->rowptr.p, (int32_t*)p->d_l.p,
                      PlanBufs{&p->heavy_rows, &p->heavy_slot_off, &p->slot_row, &p->slot_seg, &p->row_order,
                               &p->row_desc},
                      d_stat + 3, &n_heavy, &n_slots));
    // 8. halo-1: transpose CSR + its plan (the backward aggregations, R33).  Stable radix sort
    // of (column, source row) over edges listed row by row -> each transposed row lists its
    // sources in ascending local id (deterministic).
    p->halo = halo;
    p->n_halo = n_halo;
    p->halo_pending = halo && sa && n_halo > 0;   // halo features / degrees / labels: grappa_halo_exchange
    p->t_n_heavy = p->t_n_slots = 0;
    p->t_eid_ready = halo;            // induced-core: built lazily by the first GAT backward
    p->tma.ready = p->t_tma.ready = false;   // TMA SpMM plans: rebuilt on first use
    if (halo) {
        // cub's radix sort takes an int item count
        if (nnz >= ((int64_t)1 << 31)) {
            set_error("grappa_repartition_ex: halo-1 transpose of %lld local edges exceeds the 2^31 sort limit",
                      (long long)nnz);
            return fail(GRAPPA_E_SUPPORT);
        }
        RP_TRY(p->t_rowptr.grow((size_t)(n_local + 1) * 8));
        RP_TRY(p->t_col.grow((size_t)(nnz > 0 ? nnz : 1) * 4));
        RP_TRY(p->t_deg.grow((size_t)n_local * 4));
        int end_bit = 1;
        while (((int64_t)1 << end_bit) <= n_local) end_bit++;
        size_t sort_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                        (const int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0, end_bit, s);
        const size_t e4 = al((size_t)(nnz > 0 ? nnz : 1) * 4);
        RP_TRY(p->t_tmp.grow(3 * e4 + sort_bytes));
        RP_TRY(p->t_eid.grow((size_t)(nnz > 0 ? nnz : 1) * 4));
        int32_t* erow = (int32_t*)p->t_tmp.p;
        int32_t* skeys = (int32_t*)((char*)p->t_tmp.p + e4);
        int32_t* iota = (int32_t*)((char*)p->t_tmp.p + 2 * e4);
        void* stmp = (char*)p->t_tmp.p + 3 * e4;
        if (nnz > 0) {
            k_edge_rows<<<tgrid, 256, 0, s>>>(n_core, (int64_t*)p->rowptr.p, erow);
            GRAPPA_LAUNCHED(ctx);
            k_iota<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4096), 256, 0, s>>>(nnz, iota);
            GRAPPA_LAUNCHED(ctx);
            // stable sort of edge ids by column: t_eid = forward edge of each transposed entry
            GRAPPA_CUDA(cub::DeviceRadixSort::SortPairs(stmp, sort_bytes, (const int32_t*)p->col.p, skeys,
                                                        (const int32_t*)iota, (int32_t*)p->t_eid.p, (int)nnz, 0,
                                                        end_bit, s));
            ctx->launches++;
            k_take<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4096), 256, 0, s>>>(
                nnz, (const int32_t*)p->t_eid.p, erow, (int32_t*)p->t_col.p);
            GRAPPA_LAUNCHED(ctx);
        }
        k_t_rowptr<<<(unsigned)std::min<int64_t>(ceil_div(nnz + 1, 256), 4096), 256, 0, s>>>(
            n_local, nnz, skeys, (int64_t*)p->t_rowptr.p);
        GRAPPA_LAUNCHED(ctx);
        k_row_deg<<<grid, 256, 0, s>>>(n_local, (int64_t*)p->t_rowptr.p, (int32_t*)p->t_deg.p);
        GRAPPA_LAUNCHED(ctx);
        RP_TRY(build_plan(ctx, s, n_local, (int64_t*)p->t_rowptr.p, (int32_t*)p->t_deg.p,
                          PlanBufs{&p->t_heavy_rows, &p->t_heavy_slot_off, &p->t_slot_row, &p->t_slot_seg,
                                   &p->t_row_order, &p->t_row_desc},
                          d_stat + 3, &p->t_n_heavy, &p->t_n_slots));
    }
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    // algorithmic bytes (SURVEY §8(d) d.3 per core row: rowptr 8 + d_g source columns 4 d_g +
    // kept columns 4 d_l + per-row outputs 24 + the feature row read and written 2 F s)
    ps.set_bytes((double)n_core * (8.0 + 24.0 + 2.0 * (feats ? feat_dim * esz : 0)) + 4.0 * (double)sum_dg +
                 4.0 * (double)nnz);
    // publish
    grappa_part_info& I = p->info;
    I.n_core = n_local; I.nnz = nnz; I.n_seeds = n_seeds; I.base = base; I.swept = swept;
    I.n_halo = n_halo;
    I.feat_dim = feats ? feat_dim : 0; I.dtype = dtype;
    I.rowptr = (int64_t*)p->rowptr.p; I.col = (int32_t*)p->col.p;
    I.core_global = (int32_t*)p->core_global.p; I.d_l = (int32_t*)p->d_l.p; I.d_g = (int32_t*)p->d_g.p;
    I.norm_gcn = (float*)p->norm_gcn.p; I.norm_sage = (float*)p->norm_sage.p;
    I.node_w = (float*)p->node_w.p;
    I.seeds = (int32_t*)p->seeds.p; I.labels = (int32_t*)p->labels.p; I.x = p->x.p;
    I.n_heavy = n_heavy; I.n_slots = n_slots;
    I.t_rowptr = halo ? (int64_t*)p->t_rowptr.p : nullptr;
    I.t_col = halo ? (int32_t*)p->t_col.p : nullptr;
    I.c_uniform = hs.sum_r / (double)n_seeds;
    I.D = hs.D;
    const double D = (double)hs.D;
    I.c_resampling = D < 1e-9 ? 1.0 : std::min(1.0 / D, 10.0);
    I.c_resampling_hm = hs.sum_dl > 0 ? (double)hs.sum_dl / (double)hs.sum_dg : 1.0;
    *inout = p;
    return GRAPPA_OK;
#undef RP_TRY
}

extern "C" grappa_status grappa_repartition_ex(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                               int32_t feat_dim, grappa_dtype dtype,
                                               const int32_t* chunk_of, int32_t num_chunks,
                                               int32_t base, int32_t swept, const uint8_t* train_mask,
                                               const int32_t* labels, unsigned flags,
                                               grappa_part** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && g && chunk_of && train_mask && inout, GRAPPA_E_ARG,
               "grappa_repartition: null argument");
    return repart_impl(ctx, g, feats, feat_dim, dtype, chunk_of, num_chunks, base, swept, train_mask, labels,
                       flags, nullptr, nullptr, inout, (cudaStream_t)stream);
}

extern "C" grappa_status grappa_repartition_shards(grappa_ctx* ctx, const grappa_shard* base,
                                                   const grappa_shard* swept, const int32_t* chunk_of,
                                                   int64_t num_nodes, int32_t num_chunks, grappa_part** inout,
                                                   void* stream) {
    return grappa_repartition_shards_ex(ctx, base, swept, chunk_of, num_nodes, num_chunks, 0u, inout, stream);
}

extern "C" grappa_status grappa_repartition_shards_ex(grappa_ctx* ctx, const grappa_shard* base,
                                                      const grappa_shard* swept, const int32_t* chunk_of,
                                                      int64_t num_nodes, int32_t num_chunks, unsigned flags,
                                                      grappa_part** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && base && swept && chunk_of && inout, GRAPPA_E_ARG,
               "grappa_repartition_shards: null argument");
    const grappa_shard_info &A = base->info, &B = swept->info;
    GRAPPA_ARG(A.feat_dim == B.feat_dim && (A.feat_dim == 0 || A.dtype == B.dtype), GRAPPA_E_ARG,
               "grappa_repartition_shards: shards differ in feature width or dtype");
    GRAPPA_ARG(A.n_rows + B.n_rows <= num_nodes, GRAPPA_E_ARG,
               "grappa_repartition_shards: shards larger than the graph");
    // only num_nodes is read from the CSR descriptor in sharded mode (rank table over N)
    grappa_csr gn{num_nodes, 0, nullptr, nullptr};
    return repart_impl(ctx, &gn, A.feat_dim ? (const void*)A.x : nullptr, A.feat_dim, A.dtype, chunk_of,
                       num_chunks, A.chunk, B.chunk, A.train, A.labels, flags, base, swept, inout,
                       (cudaStream_t)stream);
}

// ------------------------------------------------------------------ batched switch
namespace grappa {
// split rows of a local CSR: count (d > kSegLen) and slots (sum ceil(d / kSegLen)), integers
__global__ void k_heavy_count(int64_t n, const int32_t* __restrict__ d_l, unsigned long long* out) {
    unsigned long long h = 0, sl = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = d_l[i];
        if (d > kSegLen) {
            h++;
            sl += (unsigned long long)ceil_div(d, kSegLen);
        }
    }
    h = warp_sum(h);
    sl = warp_sum(sl);
    if ((threadIdx.x & 31) == 0 && (h | sl)) {
        atomicAdd(out, h);
        atomicAdd(out + 1, sl);
    }
}
__global__ void k_chunk_hist(int64_t n, const int32_t* __restrict__ chunk_of, int C, unsigned long long* cnt) {
    __shared__ unsigned int sh[256];
    const bool loc = C <= 256;
    if (loc)
        for (int i = threadIdx.x; i < C; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = chunk_of[v];
        if (c >= 0 && c < C) {
            if (loc) atomicAdd(&sh[c], 1u);
            else atomicAdd(&cnt[c], 1ull);
        }
    }
    __syncthreads();
    if (loc)
        for (int i = threadIdx.x; i < C; i += blockDim.x)
            if (sh[i]) atomicAdd(&cnt[i], (unsigned long long)sh[i]);
}
// per-chunk sums of the nodes' global degrees (block-local shared sums for C <= 64)
__global__ void k_chunk_deg(int64_t n, const int32_t* __restrict__ chunk_of, const int64_t* __restrict__ rowptr,
                            int C, unsigned long long* sum) {
    __shared__ unsigned long long sh[64];
    const bool loc = C <= 64;
    if (loc)
        for (int i = threadIdx.x; i < C; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = chunk_of[v];
        const unsigned long long d = (unsigned long long)(rowptr[v + 1] - rowptr[v]);
        if (c >= 0 && c < C && d) atomicAdd(loc ? &sh[c] : &sum[c], d);
    }
    __syncthreads();
    if (loc)
        for (int i = threadIdx.x; i < C; i += blockDim.x)
            if (sh[i]) atomicAdd(&sum[i], sh[i]);
}
__global__ void k_edge_chunk(int64_t nnz, const int32_t* __restrict__ col, const int32_t* __restrict__ chunk_of,
                             uint8_t* __restrict__ ec) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        ec[e] = (uint8_t)__ldg(chunk_of + __ldg(col + e));
}
struct WriteRankOnly {
    int32_t* rank;
    __device__ void operator()(int64_t v, int64_t p, int32_t f) const { rank[v] = f ? (int32_t)p : -1; }
    __device__ void finish(int64_t, int64_t) const {}
};
}  // namespace grappa

// The switch's partitions extracted with two host syncs in total instead of five per partition:
// phase A (every partition): rank table, task split + kept counts, task offsets, per-row
// finalize (rowptr, degrees, norms, node weights, labels), seeds, split-row counts -- sizes stay
// on the device; one sync reads them all; phase B (every partition): rank table again (cheap:
// 8 bytes per node), stable fill of the local columns, features, coverage statistics, SpMM plan
// with the now-known split-row sizes; one final sync publishes the statistics.  Core sizes come
// from the caller's chunk sizes (grappa_partition's output), checked against the device counts.
extern "C" grappa_status grappa_index_create(grappa_ctx* ctx, const grappa_csr* g, const int32_t* chunk_of,
                                             int32_t num_chunks, grappa_index** out, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && g && chunk_of && out, GRAPPA_E_ARG, "grappa_index_create: null argument");
    GRAPPA_ARG(num_chunks >= 2 && num_chunks <= 255, GRAPPA_E_ARG, "grappa_index_create: need 2 <= C <= 255");
    GRAPPA_ARG(g->num_nodes > 0 && g->num_nodes < (1ll << 31) && g->nnz >= 0, GRAPPA_E_ARG,
               "grappa_index_create: num_nodes out of int32 range");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = g->num_nodes;
    grappa_index* ix = new grappa_index();
    auto fail = [&](grappa_status st) {
        grappa_index_destroy(ix);
        return st;
    };
#define IX_TRY(expr)                          \
    do {                                      \
        grappa_status _s = (expr);            \
        if (_s != GRAPPA_OK) return fail(_s); \
    } while (0)
    IX_TRY(ix->ec.grow((size_t)(g->nnz > 0 ? g->nnz : 1)));
    if (g->nnz > 0) {
        k_edge_chunk<<<(unsigned)std::min<int64_t>(ceil_div(g->nnz, 256), (int64_t)ctx->sm_count * 32), 256, 0, s>>>(
            g->nnz, g->col, chunk_of, (uint8_t*)ix->ec.p);
        GRAPPA_LAUNCHED(ctx);
    }
    IX_TRY(ctx->small.grow((size_t)num_chunks * 16));
    unsigned long long* d_cnt = (unsigned long long*)ctx->small.p;
    if (cudaMemsetAsync(d_cnt, 0, (size_t)num_chunks * 16, s) != cudaSuccess) return fail(GRAPPA_E_CUDA);
    const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(N, 256), (int64_t)ctx->sm_count * 8));
    k_chunk_hist<<<gr, 256, 0, s>>>(N, chunk_of, num_chunks, d_cnt);
    GRAPPA_LAUNCHED(ctx);
    k_chunk_deg<<<gr, 256, 0, s>>>(N, chunk_of, g->rowptr, num_chunks, d_cnt + num_chunks);
    GRAPPA_LAUNCHED(ctx);
    std::vector<int64_t> h((size_t)num_chunks * 2);
    if (cudaMemcpyAsync(h.data(), d_cnt, (size_t)num_chunks * 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("grappa_index_create: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    ix->sizes.assign(h.begin(), h.begin() + num_chunks);
    ix->degs.assign(h.begin() + num_chunks, h.end());
    ix->rowptr = g->rowptr; ix->col = g->col; ix->chunk_of = chunk_of;
    ix->N = N; ix->nnz = g->nnz; ix->C = num_chunks;
    *out = ix;
    return GRAPPA_OK;
#undef IX_TRY
}

extern "C" void grappa_index_destroy(grappa_index* ix) {
    if (!ix) return;
    ix->ec.release();
    delete ix;
}

extern "C" grappa_status grappa_index_query(const grappa_index* ix, int64_t* chunk_sizes, int64_t* chunk_degrees) {
    GRAPPA_ARG(ix, GRAPPA_E_ARG, "grappa_index_query: null argument");
    for (int c = 0; c < ix->C; c++) {
        if (chunk_sizes) chunk_sizes[c] = ix->sizes[c];
        if (chunk_degrees) chunk_degrees[c] = ix->degs[c];
    }
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_repartition_batch(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                                  int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                                  int32_t num_chunks, const int64_t* chunk_sizes, int32_t n_parts,
                                                  const int32_t* bases, const int32_t* swepts,
                                                  const uint8_t* train_mask, const int32_t* labels,
                                                  grappa_part** parts, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && g && chunk_of, GRAPPA_E_ARG, "grappa_repartition_batch: null argument");
    grappa_index* ix = nullptr;
    GRAPPA_TRY(grappa_index_create(ctx, g, chunk_of, num_chunks, &ix, stream));
    const grappa_status st = grappa_repartition_batch_ix(ctx, g, feats, feat_dim, dtype, ix, chunk_sizes, n_parts,
                                                         bases, swepts, train_mask, labels, parts, stream);
    cudaStreamSynchronize((cudaStream_t)stream);     // the index's buffer is in use until here
    grappa_index_destroy(ix);
    return st;
}

extern "C" grappa_status grappa_repartition_batch_ix(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                                     int32_t feat_dim, grappa_dtype dtype, const grappa_index* ix,
                                                     const int64_t* chunk_sizes, int32_t n_parts,
                                                     const int32_t* bases, const int32_t* swepts,
                                                     const uint8_t* train_mask, const int32_t* labels,
                                                     grappa_part** parts, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && g && ix && chunk_sizes && bases && swepts && train_mask && parts && n_parts >= 1,
               GRAPPA_E_ARG, "grappa_repartition_batch: null argument");
    GRAPPA_ARG(feats == nullptr || (feat_dim > 0 && feat_dim % 16 == 0), GRAPPA_E_SHAPE,
               "grappa_repartition_batch: feat_dim must be a positive multiple of 16");
    GRAPPA_ARG(ix->col == g->col && ix->rowptr == g->rowptr && ix->N == g->num_nodes && ix->nnz == g->nnz,
               GRAPPA_E_ARG, "grappa_repartition_batch: the index was built for another graph");
    const int32_t* chunk_of = ix->chunk_of;
    const int32_t num_chunks = ix->C;
    const int K = n_parts;
    std::vector<int64_t> ncore(K);
    for (int c = 0; c < num_chunks; c++)
        GRAPPA_ARG(ix->sizes[c] == chunk_sizes[c], GRAPPA_E_ARG,
                   "grappa_repartition_batch: chunk_sizes[%d] = %lld but the chunk map holds %lld nodes", c,
                   (long long)chunk_sizes[c], (long long)ix->sizes[c]);
    for (int k = 0; k < K; k++) {
        GRAPPA_ARG(bases[k] != swepts[k], GRAPPA_E_ARG, "grappa_repartition_batch: base == swept (S:139)");
        GRAPPA_ARG(bases[k] >= 0 && swepts[k] >= 0 && bases[k] < num_chunks && swepts[k] < num_chunks, GRAPPA_E_ARG,
                   "grappa_repartition_batch: chunk id out of range");
        ncore[k] = chunk_sizes[bases[k]] + chunk_sizes[swepts[k]];
        GRAPPA_ARG(ncore[k] > 0 && ncore[k] <= g->num_nodes, GRAPPA_E_ARG, "grappa_repartition_batch: bad chunk sizes");
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = g->num_nodes;
    const int64_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
    ProfScope ps(ctx, s, GRAPPA_K_REPART, 0.0, 0.0);
    // new partition objects (destroyed again if the batch fails)
    std::vector<grappa_part*> P(K);
    std::vector<bool> fresh(K);
    for (int k = 0; k < K; k++) {
        fresh[k] = parts[k] == nullptr;
        P[k] = parts[k] ? parts[k] : new grappa_part();
    }
    auto fail = [&](grappa_status st) {
        for (int j = 0; j < grappa_ctx::kRpStreams; j++)      // side streams may still use them
            if (ctx->rp_s[j]) cudaStreamSynchronize(ctx->rp_s[j]);
        for (int k = 0; k < K; k++)
            if (fresh[k]) grappa_part_destroy(P[k]);
        return st;
    };
#define RB_TRY(expr)                               \
    do {                                           \
        grappa_status _s = (expr);                 \
        if (_s != GRAPPA_OK) return fail(_s);      \
    } while (0)
#define RB_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            set_error("grappa_repartition_batch: %s", cudaGetErrorString(_e));          \
            return fail(GRAPPA_E_CUDA);                                                 \
        }                                                                               \
    } while (0)
    // device stats per partition: [0] n_core [1] nnz [2] n_seeds [3] n_heavy [4] n_slots [5] T
    // [6] unused [7] sum d_g ; then the partitions' SeedStats
    constexpr int kSt = 16;
    RB_TRY(ctx->small.grow((size_t)K * kSt * 8 + (size_t)K * sizeof(SeedStats)));
    int64_t* d_stat0 = (int64_t*)ctx->small.p;
    SeedStats* d_ss0 = (SeedStats*)(d_stat0 + (size_t)K * kSt);
    RB_CUDA(cudaMemsetAsync(d_stat0, 0, (size_t)K * kSt * 8, s));
    // rank table (int32 [N], read for kept edges only); membership from the per-edge chunk bytes
    // one table per partition when K of them fit in 1 GiB (phase B then reuses phase A's), else
    // one shared table recomputed in phase B
    const bool keep_ranks = (double)K * (double)N * 4.0 <= (double)(1ll << 30);
    RB_TRY(ctx->red_ws.grow((size_t)N * sizeof(int32_t) * (keep_ranks ? K : 1)));
    int32_t* rank0 = (int32_t*)ctx->red_ws.p;
    auto rank_of = [&](int k) { return keep_ranks ? rank0 + (size_t)k * N : rank0; };
    // task tables of every partition (phase B reads them): one workspace, K slices
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    std::vector<int64_t> Tmax(K);
    std::vector<size_t> ws_off(K + 1, 0);
    for (int k = 0; k < K; k++) {
        // sum over core rows of max(1, ceil(d / L)) <= n + floor(sum d / L)
        Tmax[k] = ncore[k] + (ix->degs[bases[k]] + ix->degs[swepts[k]]) / kTaskLen + 1;
        ws_off[k + 1] = ws_off[k] + al((size_t)(ncore[k] + 1) * 4) + al((size_t)Tmax[k] * 16) +
                        al((size_t)Tmax[k] * 4) + al((size_t)(Tmax[k] + 1) * 8);
    }
    RB_TRY(ctx->rp_ws.grow(ws_off[K]));
    struct TW { int32_t* off; int4* desc; int32_t* cnt; int64_t* out; };
    std::vector<TW> tw(K);
    for (int k = 0; k < K; k++) {
        char* w = (char*)ctx->rp_ws.p + ws_off[k];
        tw[k].off = (int32_t*)w; w += al((size_t)(ncore[k] + 1) * 4);
        tw[k].desc = (int4*)w; w += al((size_t)Tmax[k] * 16);
        tw[k].cnt = (int32_t*)w; w += al((size_t)Tmax[k] * 4);
        tw[k].out = (int64_t*)w;
    }
    const unsigned tgrid = (unsigned)ctx->sm_count * 16;
    const uint8_t* ec = (const uint8_t*)ix->ec.p;
    // The partitions are independent: partition k runs on side stream k % NS with its own scan
    // partials, bucket counters and (if not kept per partition) rank table, so the chains of
    // small latency-bound kernels of different partitions overlap.  Fork after the stats memset,
    // join before each host sync.
    const int NS = std::min(K, (int)grappa_ctx::kRpStreams);
    // the side streams take the caller stream's priority (a prefetched switch runs on a
    // high-priority stream so its kernels are scheduled ahead of the epoch being replayed)
    int prio = 0;
    RB_CUDA(cudaStreamGetPriority(s, &prio));
    for (int j = 0; j < NS; j++) {
        if (ctx->rp_s[j] && ctx->rp_prio != prio) {
            RB_CUDA(cudaStreamSynchronize(ctx->rp_s[j]));
            RB_CUDA(cudaStreamDestroy(ctx->rp_s[j]));
            ctx->rp_s[j] = nullptr;
        }
        if (!ctx->rp_s[j]) RB_CUDA(cudaStreamCreateWithPriority(&ctx->rp_s[j], cudaStreamNonBlocking, prio));
    }
    ctx->rp_prio = prio;
    for (int j = 0; j <= NS; j++)
        if (!ctx->rp_ev[j]) RB_CUDA(cudaEventCreateWithFlags(&ctx->rp_ev[j], cudaEventDisableTiming));
    auto fork = [&]() -> grappa_status {
        GRAPPA_CUDA(cudaEventRecord(ctx->rp_ev[NS], s));
        for (int j = 0; j < NS; j++) GRAPPA_CUDA(cudaStreamWaitEvent(ctx->rp_s[j], ctx->rp_ev[NS], 0));
        return GRAPPA_OK;
    };
    auto join = [&]() -> grappa_status {
        for (int j = 0; j < NS; j++) {
            GRAPPA_CUDA(cudaEventRecord(ctx->rp_ev[j], ctx->rp_s[j]));
            GRAPPA_CUDA(cudaStreamWaitEvent(s, ctx->rp_ev[j], 0));
        }
        return GRAPPA_OK;
    };
    if (!keep_ranks)
        for (int j = 0; j < NS; j++) RB_TRY(ctx->rp_rank[j].grow((size_t)N * sizeof(int32_t)));
    auto rank_k = [&](int k) { return keep_ranks ? rank_of(k) : (int32_t*)ctx->rp_rank[k % NS].p; };
    RB_TRY(fork());
    // ---------------------------------------------------------------- phase A
    for (int k = 0; k < K; k++) {
        cudaStream_t s = ctx->rp_s[k % NS];            // (shadows the call's stream)
        DevBuf* sws = &ctx->rp_scan[k % NS];
        grappa_part* p = P[k];
        int64_t* d_stat = d_stat0 + (size_t)k * kSt;
        const int64_t n = ncore[k];
        RB_TRY(p->core_global.grow((size_t)n * 4));
        RB_TRY(p->d_l.grow(n * 4));
        RB_TRY(p->d_g.grow(n * 4));
        RB_TRY(p->norm_gcn.grow(n * 4));
        RB_TRY(p->norm_sage.grow(n * 4));
        RB_TRY(p->node_w.grow(n * 12));
        RB_TRY(p->labels.grow(n * 4));
        RB_TRY(p->rowptr.grow((n + 1) * 8));
        RB_TRY(p->seeds.grow(n * 4));
        RB_TRY(p->heavy_rows.grow((size_t)n * 4));
        const int32_t* cg = (const int32_t*)p->core_global.p;
        RB_TRY(device_scan(ctx, FlagCore{chunk_of, bases[k], swepts[k]}, N,
                           WriteRank{rank_k(k), (int32_t*)p->core_global.p, d_stat}, s, nullptr, sws));
        unsigned grid;
        rp_grid(ctx, n, 256, &grid);
        RB_TRY(device_scan(ctx, NumTasks{cg, g->rowptr}, n, WriteTasks{tw[k].off, tw[k].desc, d_stat, cg, g->rowptr}, s,
                           nullptr, sws));
        {
            const Member mb{nullptr, ec, bases[k], swepts[k], 0};
            k_task_count<true><<<tgrid, 256, 0, s>>>(d_stat + 5, tw[k].desc, g->col, mb, tw[k].cnt);
        }
        GRAPPA_LAUNCHED(ctx);
        RB_TRY(device_scan(ctx, ReadTcount{tw[k].cnt, d_stat + 5}, Tmax[k], WriteTaskOut{tw[k].out, d_stat}, s,
                           nullptr, sws));
        k_row_finalize<<<grid, 256, 0, s>>>(n, tw[k].off, tw[k].out, cg, g->rowptr, labels, (int64_t*)p->rowptr.p,
                                             (int32_t*)p->d_l.p, (int32_t*)p->d_g.p, (float*)p->norm_gcn.p,
                                             (float*)p->norm_sage.p, (float*)p->node_w.p, n, (int32_t*)p->labels.p,
                                             (unsigned long long*)(d_stat + 7));
        GRAPPA_LAUNCHED(ctx);
        RB_TRY(device_scan(ctx, FlagSeed{cg, train_mask}, n, WriteCompact{(int32_t*)p->seeds.p, d_stat, 2}, s,
                           nullptr, sws));
        k_heavy_count<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 4)),
                        256, 0, s>>>(n, (const int32_t*)p->d_l.p, (unsigned long long*)(d_stat + 3));
        GRAPPA_LAUNCHED(ctx);
    }
    RB_TRY(join());
    std::vector<int64_t> st((size_t)K * kSt);
    RB_CUDA(cudaMemcpyAsync(st.data(), d_stat0, (size_t)K * kSt * 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < K; k++) {
        const int64_t* h = &st[(size_t)k * kSt];
        if (h[0] != ncore[k]) {
            set_error("grappa_repartition_batch: chunk_sizes disagree with chunk_of (%lld vs %lld core nodes)",
                      (long long)ncore[k], (long long)h[0]);
            return fail(GRAPPA_E_ARG);
        }
        if (h[2] == 0) {
            set_error("grappa_repartition_batch: partition (%d,%d) has no seeds (S:213)", bases[k], swepts[k]);
            return fail(GRAPPA_E_EMPTY);
        }
    }
    // ---------------------------------------------------------------- phase B
    double bytes = 0.0;
    RB_TRY(fork());
    for (int k = 0; k < K; k++) {
        cudaStream_t s = ctx->rp_s[k % NS];
        DevBuf* sws = &ctx->rp_scan[k % NS];
        grappa_part* p = P[k];
        const int64_t* h = &st[(size_t)k * kSt];
        const int64_t n = ncore[k], nnz = h[1], n_seeds = h[2], n_heavy = h[3], n_slots = h[4];
        const int32_t* cg = (const int32_t*)p->core_global.p;
        int32_t* rank = rank_k(k);
        if (!keep_ranks)
            RB_TRY(device_scan(ctx, FlagCore{chunk_of, bases[k], swepts[k]}, N, WriteRankOnly{rank}, s, nullptr, sws));
        RB_TRY(p->col.grow((size_t)(nnz > 0 ? nnz : 1) * 4));
        {
            const Member mb{nullptr, ec, bases[k], swepts[k], 0};
            k_task_fill<true><<<tgrid, 256, 0, s>>>(d_stat0 + (size_t)k * kSt + 5, tw[k].desc, tw[k].out, g->col, mb,
                                                    (int32_t*)p->col.p);
        }
        GRAPPA_LAUNCHED(ctx);
        if (nnz > 0) {
            k_relabel<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), (int64_t)ctx->sm_count * 32), 256, 0, s>>>(
                nnz, rank, (int32_t*)p->col.p);
        }
        GRAPPA_LAUNCHED(ctx);
        unsigned grid;
        rp_grid(ctx, n, 256, &grid);
        if (feats) {
            RB_TRY(p->x.grow((size_t)n * feat_dim * esz));
            k_gather_rows<<<grid, 256, 0, s>>>(n, feat_dim * esz, cg, (const uint4*)feats, (uint4*)p->x.p);
            GRAPPA_LAUNCHED(ctx);
        }
        int nb = seed_stat_blocks(ctx, n_seeds);
        if (nb < 1) nb = 1;
        // this stream's small workspace: degree-bucket counters, then the seed-statistics partials
        const size_t bins_b = (size_t)2 * kDegBuckets * 8;
        RB_TRY(ctx->rp_small[k % NS].grow(bins_b + (size_t)nb * sizeof(SeedStats)));
        unsigned long long* bins = (unsigned long long*)ctx->rp_small[k % NS].p;
        SeedStats* sp = (SeedStats*)((char*)ctx->rp_small[k % NS].p + bins_b);
        k_seed_stats<<<nb, kStatThreads, 0, s>>>(n_seeds, (int32_t*)p->seeds.p, (int32_t*)p->d_l.p,
                                                  (int32_t*)p->d_g.p, sp);
        GRAPPA_LAUNCHED(ctx);
        k_seed_stats_final<<<1, 32, 0, s>>>(nb, sp, d_ss0 + k);
        GRAPPA_LAUNCHED(ctx);
        // SpMM plan with the known split-row sizes (no sync)
        RB_TRY(build_plan_sized(ctx, s, n, (int64_t*)p->rowptr.p, (int32_t*)p->d_l.p,
                                PlanBufs{&p->heavy_rows, &p->heavy_slot_off, &p->slot_row, &p->slot_seg,
                                         &p->row_order, &p->row_desc},
                                d_stat0 + (size_t)k * kSt + 8, n_heavy, n_slots, sws, bins));
        p->halo = false;
        p->n_halo = 0;
        p->halo_pending = false;
        p->t_n_heavy = p->t_n_slots = 0;
        p->t_eid_ready = false;
        p->tma.ready = p->t_tma.ready = false;
        grappa_part_info& I = p->info;
        I = grappa_part_info{};
        I.n_core = n; I.nnz = nnz; I.n_seeds = n_seeds; I.base = bases[k]; I.swept = swepts[k];
        I.n_halo = 0;
        I.feat_dim = feats ? feat_dim : 0; I.dtype = dtype;
        I.rowptr = (int64_t*)p->rowptr.p; I.col = (int32_t*)p->col.p;
        I.core_global = (int32_t*)p->core_global.p; I.d_l = (int32_t*)p->d_l.p; I.d_g = (int32_t*)p->d_g.p;
        I.norm_gcn = (float*)p->norm_gcn.p; I.norm_sage = (float*)p->norm_sage.p;
        I.node_w = (float*)p->node_w.p;
        I.seeds = (int32_t*)p->seeds.p; I.labels = (int32_t*)p->labels.p; I.x = p->x.p;
        I.n_heavy = n_heavy; I.n_slots = n_slots;
        // algorithmic bytes (SURVEY §8(d) d.3 per core row): rowptr 8 + the d_g source columns + the
        // d_l kept columns + outputs 24 + the feature row read and written
        bytes += (double)n * (8.0 + 24.0 + 2.0 * (feats ? feat_dim * esz : 0)) + 4.0 * (double)h[7] + 4.0 * (double)nnz;
    }
    RB_TRY(join());
    std::vector<SeedStats> hs(K);
    RB_CUDA(cudaMemcpyAsync(hs.data(), d_ss0, (size_t)K * sizeof(SeedStats), cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < K; k++) {
        grappa_part_info& I = P[k]->info;
        I.c_uniform = hs[k].sum_r / (double)I.n_seeds;
        I.D = hs[k].D;
        const double D = (double)hs[k].D;
        I.c_resampling = D < 1e-9 ? 1.0 : std::min(1.0 / D, 10.0);
        I.c_resampling_hm = hs[k].sum_dl > 0 ? (double)hs[k].sum_dl / (double)hs[k].sum_dg : 1.0;
        parts[k] = P[k];
    }
    ps.set_bytes(bytes);
    return GRAPPA_OK;
#undef RB_TRY
#undef RB_CUDA
}

static grappa_status part_copy(const grappa_part* p, const grappa_part_host* h, bool to_host, cudaStream_t s) {
    const grappa_part_info& I = p->info;
    const size_t es = I.dtype == GRAPPA_BF16 ? 2 : 4;
    struct F { void* host; void* dev; size_t bytes; } f[] = {
        {h->rowptr, p->rowptr.p, (size_t)(I.n_core + 1) * 8}, {h->col, p->col.p, (size_t)I.nnz * 4},
        {h->d_l, p->d_l.p, (size_t)I.n_core * 4}, {h->norm_gcn, p->norm_gcn.p, (size_t)I.n_core * 4},
        {h->norm_sage, p->norm_sage.p, (size_t)I.n_core * 4}, {h->seeds, p->seeds.p, (size_t)I.n_seeds * 4},
        {h->labels, p->labels.p, (size_t)I.n_core * 4}, {h->x, p->x.p, (size_t)I.n_core * I.feat_dim * es},
        {h->node_w, p->node_w.p, (size_t)I.n_core * 12}};
    for (const F& x : f) {
        if (!x.host || !x.bytes) continue;
        if (to_host) GRAPPA_CUDA(cudaMemcpyAsync(x.host, x.dev, x.bytes, cudaMemcpyDeviceToHost, s));
        else GRAPPA_CUDA(cudaMemcpyAsync(x.dev, x.host, x.bytes, cudaMemcpyHostToDevice, s));
    }
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_part_download(const grappa_part* part, const grappa_part_host* dst, void* stream) {
    GRAPPA_ARG(part && dst, GRAPPA_E_ARG, "grappa_part_download: null argument");
    return part_copy(part, dst, true, (cudaStream_t)stream);
}

extern "C" grappa_status grappa_part_upload(grappa_part* part, const grappa_part_host* src, void* stream) {
    GRAPPA_ARG(part && src, GRAPPA_E_ARG, "grappa_part_upload: null argument");
    return part_copy(part, src, false, (cudaStream_t)stream);
}

extern "C" grappa_status grappa_part_query(const grappa_part* part, grappa_part_info* out) {
    GRAPPA_ARG(part && out, GRAPPA_E_ARG, "grappa_part_query: null argument");
    *out = part->info;
    return GRAPPA_OK;
}

extern "C" void grappa_part_destroy(grappa_part* p) {
    if (!p) return;
    for (grappa::DevBuf* b : {&p->rowptr, &p->col, &p->core_global, &p->d_l, &p->d_g, &p->norm_gcn,
                              &p->norm_sage, &p->node_w, &p->seeds, &p->labels, &p->x, &p->heavy_rows,
                              &p->heavy_slot_off, &p->slot_row, &p->slot_seg, &p->row_order,
                              &p->row_desc, &p->t_rowptr, &p->t_col, &p->t_deg, &p->t_heavy_rows,
                              &p->t_heavy_slot_off, &p->t_slot_row, &p->t_slot_seg, &p->t_row_order,
                              &p->t_row_desc, &p->t_tmp, &p->t_eid})
        b->release();
    delete p;
}

// ------------------------------------------------------------------ partition images
// A partition serialised into one host buffer (capacity mode: partitions parked in host memory
// between phases and streamed to the GPU per phase).  Layout: header, then
// every array at a 256-byte aligned offset, in the fixed order of part_arrays().
namespace {
constexpr uint64_t kImageMagic = 0x4752415050414931ull;   // "GRAPPAI1"
constexpr int kImageArrays = 27;
struct ImageHeader {
    uint64_t magic;
    grappa_part_info info;      // pointers are meaningless in the image
    int32_t halo;
    int64_t n_halo, t_n_heavy, t_n_slots;
    uint64_t off[kImageArrays], bytes[kImageArrays];
};
struct ArrRef { grappa::DevBuf* buf; size_t bytes; };

// (buffer, bytes) of every array of a partition with the given counts
static int part_arrays(grappa_part* p, const grappa_part_info& I, bool halo, int64_t t_n_heavy,
                       int64_t t_n_slots, ArrRef* out) {
    const size_t n = (size_t)I.n_core, nnz = (size_t)I.nnz, es = I.dtype == GRAPPA_BF16 ? 2 : 4;
    const size_t nh = (size_t)I.n_heavy, ns = (size_t)I.n_slots;
    int k = 0;
    auto add = [&](grappa::DevBuf& b, size_t bytes) { out[k++] = ArrRef{&b, bytes}; };
    add(p->rowptr, (n + 1) * 8); add(p->col, nnz * 4); add(p->core_global, n * 4); add(p->d_l, n * 4);
    add(p->d_g, n * 4); add(p->norm_gcn, n * 4); add(p->norm_sage, n * 4); add(p->node_w, n * 12);
    add(p->seeds, (size_t)I.n_seeds * 4); add(p->labels, n * 4); add(p->x, n * (size_t)I.feat_dim * es);
    add(p->heavy_rows, nh * 4); add(p->heavy_slot_off, (nh + 1) * 4); add(p->slot_row, ns * 4);
    add(p->slot_seg, ns * 4); add(p->row_order, n * 4); add(p->row_desc, n * 16);
    const size_t th = halo ? (size_t)t_n_heavy : 0, ts = halo ? (size_t)t_n_slots : 0;
    add(p->t_rowptr, halo ? (n + 1) * 8 : 0); add(p->t_col, halo ? nnz * 4 : 0); add(p->t_deg, halo ? n * 4 : 0);
    add(p->t_heavy_rows, th * 4); add(p->t_heavy_slot_off, halo ? (th + 1) * 4 : 0);
    add(p->t_slot_row, ts * 4); add(p->t_slot_seg, ts * 4); add(p->t_row_order, halo ? n * 4 : 0);
    add(p->t_row_desc, halo ? n * 16 : 0);
    add(p->t_eid, halo ? nnz * 4 : 0);
    return k;
}
}  // namespace

extern "C" size_t grappa_part_image_bytes(const grappa_part* part) {
    if (!part) return 0;
    grappa_part* p = const_cast<grappa_part*>(part);
    ArrRef a[kImageArrays];
    const int k = part_arrays(p, p->info, p->halo, p->t_n_heavy, p->t_n_slots, a);
    size_t off = al256(sizeof(ImageHeader));
    for (int i = 0; i < k; i++) off += al256(a[i].bytes);
    return off;
}

extern "C" grappa_status grappa_part_save(const grappa_part* part, void* host, size_t host_bytes, void* stream) {
    GRAPPA_ARG(part && host, GRAPPA_E_ARG, "grappa_part_save: null argument");
    const size_t need = grappa_part_image_bytes(part);
    GRAPPA_ARG(host_bytes >= need, GRAPPA_E_ARG, "grappa_part_save: %zu B < %zu B needed", host_bytes, need);
    grappa_part* p = const_cast<grappa_part*>(part);
    ArrRef a[kImageArrays];
    const int k = part_arrays(p, p->info, p->halo, p->t_n_heavy, p->t_n_slots, a);
    ImageHeader h{};
    h.magic = kImageMagic;
    h.info = p->info;
    h.halo = p->halo;
    h.n_halo = p->n_halo; h.t_n_heavy = p->t_n_heavy; h.t_n_slots = p->t_n_slots;
    size_t off = al256(sizeof(ImageHeader));
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < k; i++) {
        h.off[i] = off; h.bytes[i] = a[i].bytes;
        if (a[i].bytes)
            GRAPPA_CUDA(cudaMemcpyAsync((char*)host + off, a[i].buf->p, a[i].bytes, cudaMemcpyDeviceToHost, s));
        off += al256(a[i].bytes);
    }
    memcpy(host, &h, sizeof(h));
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_part_image_info(const void* host, grappa_part_info* out) {
    GRAPPA_ARG(host && out, GRAPPA_E_ARG, "grappa_part_image_info: null argument");
    ImageHeader h;
    memcpy(&h, host, sizeof(h));
    GRAPPA_ARG(h.magic == kImageMagic, GRAPPA_E_ARG, "grappa_part_image_info: not a partition image");
    *out = h.info;
    out->rowptr = nullptr; out->col = nullptr; out->core_global = nullptr; out->d_l = nullptr;
    out->d_g = nullptr; out->norm_gcn = nullptr; out->norm_sage = nullptr; out->seeds = nullptr;
    out->labels = nullptr; out->x = nullptr; out->node_w = nullptr; out->t_rowptr = nullptr; out->t_col = nullptr;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_part_load(grappa_part** inout, const void* host, void* stream) {
    GRAPPA_ARG(inout && host, GRAPPA_E_ARG, "grappa_part_load: null argument");
    ImageHeader h;
    memcpy(&h, host, sizeof(h));
    GRAPPA_ARG(h.magic == kImageMagic, GRAPPA_E_ARG, "grappa_part_load: not a partition image");
    grappa_part* p = *inout ? *inout : new grappa_part();
    ArrRef a[kImageArrays];
    const int k = part_arrays(p, h.info, h.halo != 0, h.t_n_heavy, h.t_n_slots, a);
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < k; i++) {
        if (!a[i].bytes) continue;
        grappa_status st = a[i].buf->grow(a[i].bytes);
        if (st != GRAPPA_OK) {
            if (!*inout) grappa_part_destroy(p);
            return st;
        }
        GRAPPA_CUDA(cudaMemcpyAsync(a[i].buf->p, (const char*)host + h.off[i], a[i].bytes, cudaMemcpyHostToDevice, s));
    }
    p->halo = h.halo != 0;
    p->halo_pending = false;
    p->n_halo = h.n_halo; p->t_n_heavy = h.t_n_heavy; p->t_n_slots = h.t_n_slots;
    p->t_eid_ready = p->halo;
    p->tma.ready = p->t_tma.ready = false;
    grappa_part_info& I = p->info;
    I = h.info;
    I.rowptr = (int64_t*)p->rowptr.p; I.col = (int32_t*)p->col.p;
    I.core_global = (int32_t*)p->core_global.p; I.d_l = (int32_t*)p->d_l.p; I.d_g = (int32_t*)p->d_g.p;
    I.norm_gcn = (float*)p->norm_gcn.p; I.norm_sage = (float*)p->norm_sage.p; I.node_w = (float*)p->node_w.p;
    I.seeds = (int32_t*)p->seeds.p; I.labels = (int32_t*)p->labels.p; I.x = p->x.p;
    I.t_rowptr = p->halo ? (int64_t*)p->t_rowptr.p : nullptr;
    I.t_col = p->halo ? (int32_t*)p->t_col.p : nullptr;
    *inout = p;
    return GRAPPA_OK;
}
