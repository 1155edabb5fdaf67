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
    // caller
    const void* X = nullptr;          // [n x width] dtype
    int width = 0;                    // elements per row (multiple of 4)
    const float* row_scale = nullptr; // rs[v] or null (1)
    const float* col_scale = nullptr; // cs[u] or null (1); also weights the self term
    int self = 0;
    int relu = 0;
    int accumulate = 0;
    const void* mask = nullptr;       // [n x width] dtype or null
    void* out = nullptr;              // [n x width] dtype
    float* partial = nullptr;         // [n_slots x width] fp32 scratch
};

grappa_status spmm(grappa_ctx* ctx, const grappa_part* part, SpmmArgs a, grappa_dtype dt,
                   cudaStream_t s);
// same kernel on an explicit CSR (a.n rows, a.nnz, a.rowptr, a.col, optional split rows);
// used for the rectangular mini-batch blocks and their transposes
grappa_status spmm_csr(grappa_ctx* ctx, SpmmArgs a, grappa_dtype dt, cudaStream_t s);

}  // namespace grappa
