// common.cuh -- shared internals of libgrappa.so (status plumbing, ctx, small device helpers).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <memory>
#include <string>
#include "../../include/grappa.h"

namespace grappa {

void set_error(const char* fmt, ...);

#define GRAPPA_ARG(cond, code, ...)              \
    do {                                         \
        if (!(cond)) {                           \
            ::grappa::set_error(__VA_ARGS__);    \
            return code;                         \
        }                                        \
    } while (0)

#define GRAPPA_CUDA(expr)                                                              \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            ::grappa::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                                cudaGetErrorString(_e));                               \
            return _e == cudaErrorMemoryAllocation ? GRAPPA_E_NOMEM : GRAPPA_E_CUDA;   \
        }                                                                              \
    } while (0)

#define GRAPPA_TRY(expr)                          \
    do {                                          \
        grappa_status _s = (expr);                \
        if (_s != GRAPPA_OK) return _s;           \
    } while (0)

// Launch bookkeeping: every kernel launch goes through LAUNCHED() so the ctx can report
// how many of its own kernels ran (bench.py's gpu_launches claim).
#define GRAPPA_LAUNCHED(ctx)                                                             \
    do {                                                                                 \
        cudaError_t _e = cudaGetLastError();                                             \
        if (_e != cudaSuccess) {                                                         \
            ::grappa::set_error("%s:%d launch: %s", __FILE__, __LINE__,                  \
                                cudaGetErrorString(_e));                                 \
            return GRAPPA_E_CUDA;                                                        \
        }                                                                                \
        if (ctx) (ctx)->launches++;                                                      \
    } while (0)

// Caller allocator (grappa_ctx_create_ex): device memory of library-owned objects comes from
// the caller's allocator (the PyTorch caching allocator in the binding), so a regrow does not
// cudaFree (which synchronises the device).  Shared by the ctx and every buffer it allocated,
// so buffers of objects that outlive the ctx are still freed through the allocator that made them.
struct Allocator {
    grappa_alloc_fn alloc = nullptr;
    grappa_free_fn free = nullptr;
    void* user = nullptr;
};

// Growable device buffer of a library-owned object.  grow() allocates through the allocator of
// the API call in progress (CallScope) on that call's stream -- or cudaMalloc when the ctx has
// none or the stream is being captured into a CUDA graph -- and release() frees through the
// allocator that made the block.  grow() only allocates when the request exceeds capacity.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    std::shared_ptr<const Allocator> al;   // null: cudaMalloc'd
    void* al_stream = nullptr;
    grappa_status grow(size_t bytes);
    void release();
};

// Per API call: the ctx's allocator and the call's stream, seen by DevBuf::grow (thread-local;
// nested calls restore the outer scope).
struct CallScope {
    std::shared_ptr<const Allocator> prev_al;
    void* prev_stream;
    CallScope(const grappa_ctx* ctx, void* stream);
    ~CallScope();
};

// Optional per-kernel-class timing (grappa_profile_*): CUDA events recorded on the launch
// stream around each class's launches, plus the algorithmic bytes / flops of the call.
struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double bytes, flops;
};

}  // namespace grappa

#include <vector>

struct grappa_ctx {
    bool profiling = false;
    std::vector<grappa::ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    int device = 0;
    int rank = 0;
    int nranks = 1;
    void* comm = nullptr;        // ncclComm_t
    int sm_count = 148;
    int64_t launches = 0;
    int* d_flag = nullptr;       // non-finite flag (device)
    grappa::DevBuf scan_ws;      // device-wide scan partials
    grappa::DevBuf red_ws;       // reductions
    grappa::DevBuf small;        // small host-visible results staging (device side)
    grappa::DevBuf rp_ws;        // repartition task tables
    grappa::DevBuf sh_ws;        // sharded repartition: merged two-shard CSR
    grappa::DevBuf xf_hdr;       // shard exchange headers
    void* h_pinned = nullptr;    // pinned host staging (64 KB)
    std::shared_ptr<const grappa::Allocator> alloc;   // caller allocator (null: cudaMalloc)
    grappa::DevBuf comm_buf;     // bf16 communication buffer of grappa_aggregate_grads
    grappa::DevBuf wimg;         // streamed-weight image of the tcgen05 NN GEMM (large K)
    grappa::DevBuf loss_ws;      // loss partial sums (kept apart from the repartition scratch)
    // side streams of the batched switch (partitions extracted concurrently) and their own
    // workspaces: scan partials, degree-bucket counters + seed-statistics partials, rank table
    static constexpr int kRpStreams = 8;
    cudaStream_t rp_s[kRpStreams] = {};
    int rp_prio = 0;             // priority the side streams were created with (the caller's)
    cudaEvent_t rp_ev[kRpStreams + 1] = {};
    grappa::DevBuf rp_scan[kRpStreams], rp_small[kRpStreams], rp_rank[kRpStreams];
    // test / A-B kernel selection (grappa_set_kernel_variant): gemm 0 = tensor cores, 1/2 = CUDA
    // cores; spmm 0 = row-group, 1 = warp per row, 2 = 8 loads in flight, 3 = natural row order;
    // pair 1 = separate GCN backward GEMMs
    int var_gemm = 0, var_spmm = 0, var_pair = 0;
    int var_gemm_stream = 0;     // tcgen05 NN weight: 0 = streamed image when <= 2 tiles per SM, 1 = always, 2 = never
    // chunk map whose per-chunk counts are known (grappa_partition, or verified once by
    // grappa_repartition_batch): the batched switch allocates from them without a sync
    const int32_t* cmap_ptr = nullptr;
    int64_t cmap_n = 0;
    std::vector<int64_t> cmap_sizes;
    int64_t comm_grad_bytes = 0;   // gradient all-reduce payload bytes (grappa_comm_bytes)
    int64_t comm_other_bytes = 0;  // every other cross-GPU byte (shard / halo exchange)
};

namespace grappa {

constexpr int kWarp = 32;
// Rows whose local degree exceeds kSegLen are split into kSegLen-edge segments processed
// by separate warps, combined in segment order by a fix-up kernel (deterministic).
constexpr int kSegLen = 256;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// RAII scope: records start/stop events around one class of launches when profiling.
struct ProfScope {
    grappa_ctx* ctx;
    cudaStream_t s;
    int idx = -1;
    ProfScope(grappa_ctx* c, cudaStream_t st, int cls, double bytes, double flops);
    ~ProfScope();
    // algorithmic bytes known only after the call has sized its outputs (repartition)
    void set_bytes(double bytes);
};

// Device-wide exclusive scans: device_scan in scan.cuh.

}  // namespace grappa
