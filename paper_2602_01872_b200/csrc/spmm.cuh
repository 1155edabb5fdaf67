// spmm.cuh -- interface of the local-CSR aggregation kernel (spmm.cu).
#pragma once
#include "part.cuh"

namespace grappa {

struct SpmmArgs {
    // filled by spmm() from the partition
    int64_t n = 0;
    int64_t nnz = 0;
    const int64_t* rowptr = nullptr;
    const int32_t* col = nullptr;
    int64_t n_slots = 0, n_heavy = 0;
    const int32_t* slot_row = nullptr;
    const int32_t* slot_seg = nullptr;
    const int32_t* heavy_rows = nullptr;
    const int32_t* heavy_slot_off = nullptr;
    const int32_t* row_order = nullptr;    // optional processing order of the rows
    const int4* row_desc = nullptr;        // optional {v, deg, e0 lo, e0 hi} in that order
    // caller
    const void* X = nullptr;          // [n x width] dtype
    const void* X_self = nullptr;     // rows of the self term if not X (node-level backward: X holds
                                      // the pre-weighted rows w_u dz_u, the self term is unweighted)
    int width = 0;                    // elements per row (multiple of 4)
    const float* row_scale = nullptr; // rs[v] or null (1)
    const float* col_scale = nullptr; // cs[u] or null (1); also weights the self term
    const float* nbr_scale = nullptr; // ns[v] or null (1): multiplies the neighbour sum only
    const float* edge_w = nullptr;    // per-edge weight w[e] (CSR order) instead of cs[u] (GAT)
    int self = 0;
    int self_sep = 0;                 // self term weighted by self_scale[v] (null: 1), not cs[v]
    const float* self_scale = nullptr;
    int relu = 0;
    int accumulate = 0;
    int64_t acc_rows = INT64_MAX;     // accumulate into out rows < acc_rows only (rows past it are
                                      // written: a block transpose's source-only rows)
    const void* mask = nullptr;       // [n x width] dtype or null
    void* out = nullptr;              // [n x width] dtype
    float* partial = nullptr;         // [n_slots x width] fp32 scratch
    int out_compact = 0;              // split rows only: write split row h to out[h] (pre-pass
                                      // of the fused kernel; no mask / accumulate / relu)
};

// TMA-gather kernel (spmm_tma.cu) for bf16 unweighted aggregations at widths 80..128; default when
// eligible (ctx variant "spmm" 0); its split rows are combined by spmm_fixup (spmm.cu)
bool spmm_tma_eligible(const grappa_ctx* ctx, const SpmmArgs& a, grappa_dtype dt);
grappa_status spmm_tma(grappa_ctx* ctx, const grappa_part* part, bool transpose, const SpmmArgs& a,
                       cudaStream_t s);
grappa_status spmm_fixup(grappa_ctx* ctx, const SpmmArgs& a, cudaStream_t s);

grappa_status spmm(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                   cudaStream_t s);
// the transpose operator A_loc^T (backward aggregations): A_loc itself for induced-core
// partitions (symmetric), the stored transpose for halo-1 partitions
grappa_status spmm_t(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                     cudaStream_t s);
// same kernel on an explicit CSR (a.n rows, a.nnz, a.rowptr, a.col, optional split rows);
// used for the rectangular mini-batch blocks and their transposes
grappa_status spmm_csr(grappa_ctx* ctx, SpmmArgs a, grappa_dtype dt, cudaStream_t s);
// out[v] = scale[v] * X[v] over n rows of `width` elements (rounded to dt)
grappa_status row_scale(grappa_ctx* ctx, const void* X, int64_t n, int width, const float* scale, void* out,
                        grappa_dtype dt, cudaStream_t s);

}  // namespace grappa
