// gemm.cuh -- dense feature-transform GEMMs of a4/a6 (the only dense contractions).
#pragma once
#include "common.cuh"

namespace grappa {

// C = [A1 | A2] * op(B), fp32 accumulate.
//   A1 [M x K1], A2 [M x K2] (dtype, row-major; A2 may be null with K2 = 0)
//   B fp32: b_trans = 0 -> [K x N] row-major;  b_trans = 1 -> [N x K] row-major (i.e. W^T)
//   columns [0, n_split) -> C1 (row stride n_split), [n_split, N) -> C2 (stride N - n_split)
//   epilogue on C1 columns: *= row_scale[m] (if set),
//   *= 1[mask > 0] (mask [M x n_split], dtype), then ReLU if relu.
struct GemmArgs {
    int64_t M = 0;
    int K1 = 0, K2 = 0, N = 0;
    const void* A1 = nullptr;
    const void* A2 = nullptr;
    const float* B = nullptr;
    int b_trans = 0;
    int relu = 0;
    const void* mask = nullptr;
    int n_split = 0;
    void* C1 = nullptr;
    void* C2 = nullptr;
    const float* row_scale = nullptr;
};

// dW = [A1 | A2]^T * B  ([K1+K2] x N, fp32), reduction over the M rows split into slabs
// whose fp32 partials (ws) are summed in slab order (deterministic split-K).
struct GemmTNArgs {
    int64_t M = 0;
    int K1 = 0, K2 = 0, N = 0;
    const void* A1 = nullptr;
    const void* A2 = nullptr;
    const void* B = nullptr;  // [M x N] dtype
    float* C = nullptr;       // [(K1+K2) x N] fp32
    float* ws = nullptr;      // split-K partials
};

constexpr int kMaxSplitK = 256;
// fp32 CUDA-core kernels (gemm_f32.cu)
bool sgemm_supported(int K1, int K2, int N);
grappa_status sgemm_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s);
grappa_status sgemm_tn_partials(grappa_ctx* ctx, const GemmTNArgs& g, int slabs, int64_t rps, cudaStream_t s);
// workspace for gemm_tn (max over the SIMT and tcgen05 plans); K = K1 + K2
size_t gemm_tn_ws_bytes(int64_t M, int K1, int K2, int N);

// dispatch: bf16 storage -> tcgen05 kernels (gemm_tc.cu) when the shape fits, else SIMT
grappa_status gemm_nn(grappa_ctx* ctx, const GemmArgs& g, grappa_dtype dt, cudaStream_t s);
grappa_status gemm_tn(grappa_ctx* ctx, const GemmTNArgs& g, grappa_dtype dt, cudaStream_t s);

// tcgen05 implementations (bf16 operands, fp32 TMEM accumulators)
bool gemm_tc_nn_supported(const GemmArgs& g);
bool gemm_tc_tn_supported(const GemmTNArgs& g);
grappa_status gemm_tc_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s);
grappa_status gemm_tc_tn(grappa_ctx* ctx, const GemmTNArgs& g, cudaStream_t s);
size_t gemm_tc_tn_ws_bytes(int64_t M, int K1, int K2, int N);
// GCN backward pair in one pass over dT and h_in (bf16, tcgen05): dz_in = (dT W^T) * relu'(h_in)
// [* rs] and dW = h_in^T dT (partials in ws, summed in CTA order).  f_in in (64, 128], f_out <= 128.
bool gemm_tc_pair_supported(int64_t M, int f_in, int f_out);
grappa_status gemm_tc_pair(grappa_ctx* ctx, int64_t M, int f_in, int f_out, const void* dT, const void* h,
                           const float* W, const float* rs, int gate, void* dz_in, float* ws, float* dw,
                           cudaStream_t s);
// split-fp32 tcgen05 NN for fp32 storage (3 bf16 MMAs per K step; gemm_tc.cu)
bool gemm_x3_nn_supported(const GemmArgs& g);
grappa_status gemm_x3_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s);
bool gemm_x3_tn_supported(const GemmTNArgs& g);
grappa_status gemm_x3_tn(grappa_ctx* ctx, const GemmTNArgs& g, cudaStream_t s);
// force the SIMT kernels even for bf16 (tests cross-check the two implementations)

}  // namespace grappa
