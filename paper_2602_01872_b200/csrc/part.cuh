// part.cuh -- library-owned partition object (local CSR + per-node arrays + split rows).
#pragma once
#include "common.cuh"

namespace grappa {
// dst[i] = src[idx[i]] for i < n (rows of row_bytes, a multiple of 16); warp per row
__global__ void k_gather_rows(int64_t n, int64_t row_bytes, const int32_t* __restrict__ idx,
                              const uint4* __restrict__ src, uint4* __restrict__ dst);
// softmax-CE over explicit seed rows (loss.cu)
grappa_status loss_rows(grappa_ctx* ctx, int64_t n_seeds, const int32_t* rows, const int32_t* lidx,
                        const int32_t* labels, int64_t n_rows, const void* logits, int K, int k_pad,
                        void* dlogits, double* loss_dev, grappa_dtype dtype, cudaStream_t s,
                        const float* rscale = nullptr);
// sharded repartition (shard.cu): merge two chunk shards into one CSR in local order (row i =
// core row i, rank[] = the chunk-pair rank table); features / labels / train flags follow
grappa_status shard_merge(grappa_ctx* ctx, const grappa_shard* sa, const grappa_shard* sb, const int32_t* rank,
                          int64_t n_core, int64_t* m_src, int32_t* m_deg, int64_t* m_rowptr, int32_t* m_col,
                          int32_t* m_lab, uint8_t* m_tr, void* x_out, int64_t row_bytes, int64_t* d_stat,
                          cudaStream_t s);
}  // namespace grappa

namespace grappa {
// TMA-gather SpMM plan of one operator (spmm_tma.cu): the degree-ordered 16-row tiles of the
// SpMM's row space (split-row segments, then rows by descending degree) assigned round-robin to
// `grid` persistent CTAs and stored CTA-major, so each CTA streams one contiguous range of
// "steps" (a step = one gathered row per tile row: the self row, then the j-th neighbour).
struct TmaPlan {
    DevBuf tsteps;      // int32 [grid * tpc]   steps of each tile (0 for padding tiles)
    DevBuf toff;        // int64 [grid * tpc + 1] exclusive scan of tsteps
    DevBuf tinfo;       // int2  [grid * tpc * 16] per tile row {out row | slot flag, degree}
    DevBuf stream;      // int32 [sum tsteps * 16] gather row ids, step-major
    int grid = 0;
    int64_t tpc = 0;    // tiles per CTA
    bool ready = false;
};
}  // namespace grappa

// switch index of (global CSR, chunk map): per-edge chunk bytes and per-chunk counts / degree sums
struct grappa_index {
    const int64_t* rowptr = nullptr;
    const int32_t* col = nullptr;
    const int32_t* chunk_of = nullptr;
    int64_t N = 0, nnz = 0;
    int32_t C = 0;
    grappa::DevBuf ec;                 // uint8 [nnz]: chunk_of[col[e]]
    std::vector<int64_t> sizes, degs;  // per chunk: nodes, sum of their global degrees
};

// one chunk's rows (sharded mode): ids ascending, local rowptr from 0, global neighbour ids
struct grappa_shard {
    grappa_shard_info info{};
    grappa::DevBuf ids, rowptr, col, x, labels, train;
};

struct grappa_part {
    grappa_part_info info{};
    grappa::DevBuf rowptr, col, core_global, d_l, d_g, norm_gcn, norm_sage, seeds, labels, x;
    // node-level estimator weights (R30): [w | w*norm_gcn | w*norm_sage], 3 x n_core fp32
    grappa::DevBuf node_w;
    // SpMM row splitting (rows with d_l > kSegLen): every segment of a split row is one
    // "slot" task (row, segment); slot_off gives each split row's first slot.
    grappa::DevBuf heavy_rows, heavy_slot_off, slot_row, slot_seg;
    // SpMM processing order: rows bucketed by descending local degree, so the row groups that
    // share a warp have similar trip counts (results do not depend on the order)
    grappa::DevBuf row_order;
    // per row in that order: {v, d_l, rowptr[v] lo, hi} -- one coalesced 16-byte load replaces
    // the dependent row_order -> rowptr lookups at the head of every SpMM row
    grappa::DevBuf row_desc;
    // halo-1 mode (R33): the local operator is not symmetric, so the backward aggregations run
    // on its transpose, with the same SpMM plan structures (split rows, order, descriptors)
    bool halo = false;
    int64_t n_halo = 0;
    // sharded halo-1 partition whose halo rows (features, global degree, label, node weight)
    // still have to arrive from their chunks' owners (grappa_halo_exchange)
    bool halo_pending = false;
    grappa::DevBuf t_rowptr, t_col, t_deg, t_heavy_rows, t_heavy_slot_off, t_slot_row, t_slot_seg,
        t_row_order, t_row_desc, t_tmp;
    int64_t t_n_heavy = 0, t_n_slots = 0;
    // forward edge id of every transposed entry (GAT backward needs the attention coefficient of
    // (v -> u) while walking u's transposed row): built at repartition in halo-1 mode, lazily
    // (k_gat_rev) on the first GAT backward in induced-core mode
    grappa::DevBuf t_eid;
    bool t_eid_ready = false;
    // TMA-gather SpMM plans (built on first use; invalidated by repartition / image load)
    grappa::TmaPlan tma, t_tma;
};
