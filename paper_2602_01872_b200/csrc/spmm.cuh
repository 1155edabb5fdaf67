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
    const void* mask = nullptr;       // [n x width] dtype or null
    void* out = nullptr;              // [n x width] dtype
    float* partial = nullptr;         // [n_slots x width] fp32 scratch
    int out_compact = 0;              // split rows only: write split row h to out[h] (pre-pass
                                      // of the fused kernel; no mask / accumulate / relu)
};

// Fused aggregate -> transform (bf16, tcgen05):
//   out[v] = epi( agg(X)[v] @ B ),  agg(X)[v] = rs[v] (self cs[v] X[v] + sum_u cs[u] X[u])
//   B = W [K x N] (or W^T when b_trans, W stored [N x K]), epi = relu? / relu'(mask[v]) gate,
//   agg_out (optional) receives agg(X) itself.  Same arithmetic as spmm() followed by
//   gemm_nn() except that the aggregate is rounded to bf16 once, before the transform.
struct AggMMArgs {
    const void* X = nullptr;          // [n x K] bf16
    int K = 0;
    const float* row_scale = nullptr;
    const float* col_scale = nullptr;
    int self = 0;
    const float* W = nullptr;         // fp32 master weights
    int N = 0;
    int b_trans = 0;
    int relu = 0;
    const void* mask = nullptr;       // [n x N] bf16 or null
    void* out = nullptr;              // [n x N] bf16
    void* agg_out = nullptr;          // [n x K] bf16 or null
    void* hagg = nullptr;             // scratch [n_heavy x K] bf16
    float* partial = nullptr;         // scratch [n_slots x K] fp32
};
bool spmm_mm_supported(const grappa_part* part, int K, int N, grappa_dtype dt);
grappa_status spmm_mm(grappa_ctx* ctx, const grappa_part* part, const AggMMArgs& m, cudaStream_t s);
void spmm_set_fuse(int v);
void spmm_set_wide(int v);

grappa_status spmm(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                   cudaStream_t s);
// the transpose operator A_loc^T (backward aggregations): A_loc itself for induced-core
// partitions (symmetric), the stored transpose for halo-1 partitions
grappa_status spmm_t(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                     cudaStream_t s);
// same kernel on an explicit CSR (a.n rows, a.nnz, a.rowptr, a.col, optional split rows);
// used for the rectangular mini-batch blocks and their transposes
grappa_status spmm_csr(grappa_ctx* ctx, SpmmArgs a, grappa_dtype dt, cudaStream_t s);

}  // namespace grappa
