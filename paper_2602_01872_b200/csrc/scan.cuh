// scan.cuh -- device-wide exclusive scan (reduce-then-scan, 3 kernels) built on warp scans.
// Used by the repartition (rank table, local rowptr, seed list, split-row slots).
// Deterministic: integer arithmetic only.
#pragma once
#include "common.cuh"

namespace grappa {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of one int64 per thread; returns the exclusive prefix and the
// block total in *total.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
    constexpr int NW = kScanThreads / kWarp;
    __shared__ int64_t warp_tot[NW];
    __shared__ int64_t blk_tot;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < NW ? warp_tot[lane] : 0;
        int64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < NW) warp_tot[lane] = wi - w;   // exclusive warp offsets
        if (lane == NW - 1) blk_tot = wi;
    }
    __syncthreads();
    int64_t excl = warp_tot[wid] + incl - v;
    if (total) *total = blk_tot;
    __syncthreads();
    return excl;
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(F f, int64_t n, int64_t* part) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++)
        if (base + k < n) s += f(base + k);
    int64_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Single-block exclusive scan of part[0..nb) in place; part[nb] = grand total.
__global__ void __launch_bounds__(kScanThreads) k_scan_partials(int64_t* part, int64_t nb);

template <class F, class W>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(F f, int64_t n, const int64_t* part,
                                                            W w) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t vals[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        vals[k] = (base + k < n) ? f(base + k) : 0;
        s += vals[k];
    }
    int64_t p = block_exclusive_scan(s, nullptr) + part[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) w(base + k, p, vals[k]);
        p += vals[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) w.finish(n, part[gridDim.x]);
}

// Exclusive scan of f(0..n) with per-element writer w(i, prefix, value) and w.finish(n, total).
// Grand total left in device memory at *d_total_out (pointer into ctx scratch) if requested.
// ws: partials buffer (default ctx->scan_ws; a caller on its own stream passes its own).
template <class F, class W>
grappa_status device_scan(grappa_ctx* ctx, F f, int64_t n, W w, cudaStream_t s,
                          const int64_t** d_total_out = nullptr, DevBuf* ws = nullptr) {
    int64_t nb = n > 0 ? ceil_div(n, kScanTile) : 1;
    DevBuf& buf = ws ? *ws : ctx->scan_ws;
    GRAPPA_TRY(buf.grow((size_t)(nb + 1) * sizeof(int64_t)));
    int64_t* part = (int64_t*)buf.p;
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(f, n, part);
    GRAPPA_LAUNCHED(ctx);
    k_scan_partials<<<1, kScanThreads, 0, s>>>(part, nb);
    GRAPPA_LAUNCHED(ctx);
    k_scan_down<<<(unsigned)nb, kScanThreads, 0, s>>>(f, n, part, w);
    GRAPPA_LAUNCHED(ctx);
    if (d_total_out) *d_total_out = part + nb;
    return GRAPPA_OK;
}

}  // namespace grappa
