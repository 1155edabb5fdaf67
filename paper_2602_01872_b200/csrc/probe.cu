// probe.cu -- roofline probes: the measured ceilings the bench divides its kernels by.
//
// MEASURED_PEAKS.json gives the HBM copy bandwidth and the bf16 tensor peak; the SpMM of a4/a6
// is neither: its gathered feature table (157 MB bf16 on a products partition) mostly hits the
// 126 MB L2, so its binding ceiling is the L2 (LTS) throughput for 16-byte gathers of whole
// rows.  These probes measure, live and on the same GPU:
//   HBM_COPY   dst = src over `bytes` (>> L2): (read + write) bytes / time
//   L2_READ    repeated coalesced 16-byte reads of an L2-resident buffer of `bytes`
//   L2_GATHER  the SpMM's access pattern with nothing else: groups of row_bytes/16 lanes each
//              gather whole rows of a `bytes`-sized table at hashed random row ids, 8 rows in
//              flight per lane (bytes gathered / time); with bytes < L2 this is the L2 ceiling
//              of a row gather, the roofline the SpMM's algorithmic GB/s is reported against.
// Diagnostics only: nothing of the method runs here.
#include "common.cuh"

namespace grappa {

__global__ void k_probe_copy(int64_t n16, const uint4* __restrict__ src, uint4* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_probe_read(int64_t n16, int passes, const uint4* __restrict__ src, uint32_t* __restrict__ sink) {
    uint32_t acc = 0;
    for (int p = 0; p < passes; p++)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
             i += (int64_t)gridDim.x * blockDim.x) {
            const uint4 v = __ldcg(src + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x9e3779b9u) sink[0] = acc;     // never true in practice; keeps the loads alive
}

__device__ __forceinline__ uint32_t probe_hash(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return (uint32_t)(x ^ (x >> 31));
}

__global__ void k_probe_idx(int64_t n, uint32_t n_rows, int32_t* __restrict__ idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        idx[i] = (int32_t)(probe_hash((uint64_t)i) % n_rows);
}

// G lanes per row (G = row_bytes / 16 <= 32), 32/G rows per warp, U rows in flight per lane;
// the row ids come from an index array (as the SpMM's column indices do)
template <int U>
__global__ void __launch_bounds__(256) k_probe_gather(int64_t n_gathers, int G, const int32_t* __restrict__ idx,
                                                      const uint4* __restrict__ table, uint32_t* __restrict__ sink) {
    const int lane = threadIdx.x & 31;
    const int P = 32 / G;
    const int slot = lane / G, sub = lane - slot * G;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    if (slot < P) {
        for (int64_t g0 = (warp * P + slot) * U; g0 + U <= n_gathers; g0 += warps * P * U) {
            int r[U];
#pragma unroll
            for (int u = 0; u < U; u++) r[u] = __ldg(idx + g0 + u);
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++) v[u] = __ldg(table + (int64_t)r[u] * G + sub);
#pragma unroll
            for (int u = 0; u < U; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

}  // namespace grappa

using namespace grappa;

extern "C" grappa_status grappa_roofline_probe(grappa_ctx* ctx, int kind, int64_t bytes, int32_t row_bytes,
                                               int32_t iters, double* gbps, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && gbps, GRAPPA_E_ARG, "grappa_roofline_probe: null argument");
    GRAPPA_ARG(kind >= GRAPPA_PROBE_HBM_COPY && kind <= GRAPPA_PROBE_L2_GATHER, GRAPPA_E_ARG,
               "grappa_roofline_probe: unknown kind %d", kind);
    GRAPPA_ARG(bytes >= (1 << 20) && bytes % 16 == 0 && iters >= 1, GRAPPA_E_ARG,
               "grappa_roofline_probe: bytes must be a multiple of 16 and >= 1 MiB, iters >= 1");
    GRAPPA_ARG(kind != GRAPPA_PROBE_L2_GATHER || (row_bytes >= 16 && row_bytes <= 512 && row_bytes % 16 == 0 &&
                                                 32 % (row_bytes / 16) == 0),
               GRAPPA_E_ARG, "grappa_roofline_probe: row_bytes must be 16 * a divisor of 32");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n16 = bytes / 16;
    void* a = nullptr;
    void* b = nullptr;
    uint32_t* sink = nullptr;
    int32_t* idx = nullptr;
    const int64_t n_rows = kind == GRAPPA_PROBE_L2_GATHER ? bytes / row_bytes : 0;
    const int64_t n_gathers = n_rows * 8;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    grappa_status st = GRAPPA_OK;
    double moved = 0;
    float ms = 0.f;
    const unsigned grid = (unsigned)ctx->sm_count * 8;
    auto launch = [&]() -> grappa_status {
        if (kind == GRAPPA_PROBE_HBM_COPY) {
            k_probe_copy<<<grid, 256, 0, s>>>(n16, (const uint4*)a, (uint4*)b);
        } else if (kind == GRAPPA_PROBE_L2_READ) {
            k_probe_read<<<grid, 256, 0, s>>>(n16, 8, (const uint4*)a, sink);
        } else {
            k_probe_gather<8><<<grid, 256, 0, s>>>(n_gathers, row_bytes / 16, idx, (const uint4*)a, sink);
        }
        GRAPPA_LAUNCHED(ctx);
        return GRAPPA_OK;
    };
    do {
        if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&sink, 64) != cudaSuccess ||
            (kind == GRAPPA_PROBE_HBM_COPY && cudaMalloc(&b, bytes) != cudaSuccess) ||
            (n_gathers && cudaMalloc(&idx, n_gathers * 4) != cudaSuccess)) {
            set_error("grappa_roofline_probe: cannot allocate %lld bytes", (long long)bytes);
            st = GRAPPA_E_NOMEM;
            break;
        }
        cudaMemsetAsync(a, 0x5a, bytes, s);
        if (n_gathers) {
            k_probe_idx<<<grid, 256, 0, s>>>(n_gathers, (uint32_t)n_rows, idx);
            GRAPPA_LAUNCHED(ctx);
        }
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        if ((st = launch()) != GRAPPA_OK) break;          // warm-up (and fills L2 for the L2 kinds)
        cudaEventRecord(e0, s);
        for (int i = 0; i < iters && st == GRAPPA_OK; i++) st = launch();
        cudaEventRecord(e1, s);
        if (st != GRAPPA_OK) break;
        if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) {
            set_error("grappa_roofline_probe: %s", cudaGetErrorString(cudaGetLastError()));
            st = GRAPPA_E_CUDA;
            break;
        }
        const double per = kind == GRAPPA_PROBE_HBM_COPY ? 2.0 * bytes
                           : kind == GRAPPA_PROBE_L2_READ ? 8.0 * bytes
                                                          : (double)(n_gathers / 8 * 8) * row_bytes;
        moved = per * iters;
    } while (0);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaStreamSynchronize(s);
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (sink) cudaFree(sink);
    if (idx) cudaFree(idx);
    if (st == GRAPPA_OK) *gbps = ms > 0 ? moved / (ms * 1e-3) / 1e9 : 0.0;
    return st;
}
