// sample.cu -- a10: isolated mini-batch sampling + one SAGE mini-batch step on the blocks.
//
// PAPER: P:139/P:177 (§3.2 sampling mode: k-hop subgraphs drawn from the local partition only,
// no remote reads), P:382 (Alg. 1 isolated_sampling), P:489 (B = 1000, fanouts {15,10,5}).
// SPEC S:196-222.  Readings R23-R28 (see include/grappa.h).
//
// Per hop, all on the device (one host sync per batch, at the end, to size the layer calls):
//   k_pick_floyd  thread per target: if d_l <= f take every neighbour, else f distinct
//                 positions by Floyd's algorithm (R24), O(f) whatever the degree
//   frontier      bitmap over the partition (picks marked by k_pick_floyd, targets cleared), word-popcount
//                 scan -> new sources in ascending local id; `where` maps local id -> position
//   block CSR     rowptr = scan of pick counts; each target's positions sorted ascending
//   transpose     stable radix sort of (source position, target) pairs -> CSC for backward
#include <cub/device/device_radix_sort.cuh>

#include <cstring>
#include <vector>

#include "gemm.cuh"
#include "part.cuh"
#include "scan.cuh"
#include "spmm.cuh"

namespace grappa {

constexpr int kMaxLayers = 8;
constexpr int kMaxFanout = 32;   // P:489 fanouts {25,10}, {20,15,10,5}; kernels instantiated for <=16 and <=32

__device__ __forceinline__ uint64_t smix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t hmix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Per-call parameters of grappa_sample_async, written by the host into pinned memory and copied
// to the device by the call itself, so that the call's launch sequence is identical from batch to
// batch and can be replayed as a CUDA graph (the batch index and epoch only enter the hop keys,
// the seed slice only enters k_sample_prep).
struct SampleParams {
    int64_t n_batch;
    const int32_t* batch;
    uint64_t key[kMaxLayers];   // h(seed, epoch, batch, hop) per hop
    // the partition the batch is drawn from (parameters too, so one recorded sequence serves
    // every partition whose size fits the buffers: the phases of an epoch cycle through them)
    const int64_t* rowptr;
    const int32_t* col;
    const int32_t* gid;
    const int32_t* d_l;
    const int32_t* d_g;
};
// R24: per target, f distinct local neighbour positions by Floyd's algorithm -- for j = d-f .. d-1
// draw t = floor(h(key0, gid(v), j) (j+1) / 2^64) uniform on [0, j] and keep t, or j if t is
// already kept: every f-subset equally likely (uniform without replacement), O(f) work per
// target whatever its degree (a hub costs what a leaf costs; the earlier hash-priority draw
// hashed every neighbour).  One thread per target; picks in draw order (k_fill_block sorts).
// The picked neighbours are also marked in the frontier bitmap here (cleared beforehand), which
// saves the separate marking pass over the picks.
template <int MAXF>
__global__ void k_pick_floyd(const int64_t* __restrict__ d_nt, const int32_t* __restrict__ targets,
                             const SampleParams* __restrict__ P, int f, int hop,
                             int32_t* __restrict__ picks, int32_t* __restrict__ cnt, uint32_t* __restrict__ bitmap) {
    const int64_t nt = *d_nt;
    const uint64_t key0 = P->key[hop];
    const int64_t* __restrict__ rowptr = P->rowptr;
    const int32_t* __restrict__ col = P->col;
    const int32_t* __restrict__ gid = P->gid;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = targets[t];
        const int64_t e0 = rowptr[v], d = rowptr[v + 1] - e0;
        int32_t* out = picks + t * f;
        if (d <= f) {
            for (int i = 0; i < (int)d; i++) {
                const int32_t u = col[e0 + i];
                out[i] = u;
                atomicOr(&bitmap[u >> 5], 1u << (u & 31));
            }
            cnt[t] = (int)d;
            continue;
        }
        const uint64_t kv = key0;
        const uint64_t gv = (uint64_t)gid[v];
        int64_t kept[MAXF];
#pragma unroll
        for (int k = 0; k < MAXF; k++) {
            if (k >= f) break;
            const int64_t j = d - f + k;
            const uint64_t r = smix(kv ^ smix(gv ^ smix((uint64_t)j)));
            int64_t pos = (int64_t)__umul64hi(r, (uint64_t)(j + 1));
            bool dup = false;
#pragma unroll
            for (int q = 0; q < MAXF; q++)
                if (q < k && kept[q] == pos) dup = true;
            if (dup) pos = j;
            kept[k] = pos;
        }
        // neighbour ids of the kept positions (independent loads, issued together)
        int32_t u[MAXF];
#pragma unroll
        for (int k = 0; k < MAXF; k++)
            if (k < f) u[k] = col[e0 + kept[k]];
#pragma unroll
        for (int k = 0; k < MAXF; k++)
            if (k < f) {
                out[k] = u[k];
                atomicOr(&bitmap[u[k] >> 5], 1u << (u[k] & 31));
            }
        cnt[t] = f;
    }
}

__global__ void k_unmark(const int64_t* __restrict__ d_nt, const int32_t* __restrict__ targets,
                         uint32_t* __restrict__ bitmap, int32_t* __restrict__ where, int32_t* __restrict__ src) {
    const int64_t n = *d_nt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = targets[t];
        atomicAnd(&bitmap[v >> 5], ~(1u << (v & 31)));
        where[v] = (int32_t)t;
        src[t] = v;
    }
}

struct PopWord {
    const uint32_t* w;
    __device__ int32_t operator()(int64_t i) const { return __popc(w[i]); }
};
struct WriteNew {
    const uint32_t* w; const int64_t* d_nt; int32_t* src; int32_t* where; int64_t* d_ns;
    __device__ void operator()(int64_t i, int64_t p, int32_t) const {
        uint32_t bits = w[i];
        int64_t pos = *d_nt + p;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int32_t id = (int32_t)(i * 32 + b);
            src[pos] = id;
            where[id] = (int32_t)pos;
            pos++;
        }
    }
    __device__ void finish(int64_t, int64_t total) const { *d_ns = *d_nt + total; }
};
struct CntUpTo {
    const int32_t* cnt; const int64_t* d_nt;
    __device__ int32_t operator()(int64_t t) const { return t < *d_nt ? cnt[t] : 0; }
};
struct WriteBRow {
    int64_t* rowptr; int64_t* d_nnz;
    __device__ void operator()(int64_t t, int64_t p, int32_t) const { rowptr[t] = p; }
    __device__ void finish(int64_t n, int64_t total) const { rowptr[n] = total; *d_nnz = total; }
};

// block CSR rows: positions of the picks, ascending; edge -> target id for the transpose sort
template <int MAXF>
__global__ void k_fill_block(const int64_t* __restrict__ d_nt, const int64_t* __restrict__ d_nnz,
                             int64_t cap_nnz, const int32_t* __restrict__ picks, const int32_t* __restrict__ cnt,
                             int f, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ where,
                             int32_t* __restrict__ col, int32_t* __restrict__ erow, int32_t* __restrict__ key_pad,
                             float* __restrict__ inv_cnt, const int32_t* __restrict__ targets,
                             const SampleParams* __restrict__ P, float* __restrict__ inv_cnt_node) {
    const int32_t* __restrict__ d_l = P->d_l;
    const int32_t* __restrict__ d_g = P->d_g;
    const int64_t nt = *d_nt, nnz = *d_nnz;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = cnt[t];
        int32_t p[MAXF];
#pragma unroll
        for (int j = 0; j < MAXF; j++) p[j] = j < c ? where[picks[t * f + j]] : 0x7fffffff;
#pragma unroll
        for (int a = 1; a < MAXF; a++)              // insertion sort, unrolled network
#pragma unroll
            for (int b = a; b > 0; b--)
                if (p[b] < p[b - 1]) { const int32_t x = p[b]; p[b] = p[b - 1]; p[b - 1] = x; }
        const int64_t o = rowptr[t];
        for (int j = 0; j < c; j++) { col[o + j] = p[j]; erow[o + j] = (int32_t)t; key_pad[o + j] = p[j]; }
        inv_cnt[t] = c > 0 ? 1.0f / (float)c : 0.0f;
        // node-level estimator (R30): the sampled mean times w_v = d_l/d_g (1 iff d_g = 0)
        const int32_t v = targets[t], dg = d_g[v];
        const double wv = dg == 0 ? 1.0 : (double)d_l[v] / (double)dg;
        inv_cnt_node[t] = c > 0 ? (float)(wv / (double)c) : 0.0f;
    }
    // pad the sort keys past nnz so they sort last
    for (int64_t e = nnz + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cap_nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        key_pad[e] = 0x7fffffff;
        erow[e] = 0;
    }
}

// transpose rowptr from the sorted source keys
__global__ void k_trowptr(const int64_t* __restrict__ d_ns, const int64_t* __restrict__ d_nnz,
                          const int32_t* __restrict__ skeys, int64_t* __restrict__ trowptr) {
    const int64_t ns = *d_ns, nnz = *d_nnz;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cur = e < nnz ? skeys[e] : ns;       // first source >= this edge's source
        const int64_t prev = e > 0 ? skeys[e - 1] : -1;
        for (int64_t s = prev + 1; s <= cur && s <= ns; s++) trowptr[s] = e;
    }
}

struct BatchStats {
    double sum_r, D, num, den;
};
__global__ void k_batch_stats(int n, const int32_t* seeds, const SampleParams* __restrict__ P,
                              const int64_t* brow, BatchStats* out) {
    const int32_t* d_l = P->d_l;
    const int32_t* d_g = P->d_g;
    __shared__ BatchStats sh[256];
    BatchStats a{0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int32_t v = seeds[i];
        const int l = d_l[v], g = d_g[v];
        const double s = (double)(brow[i + 1] - brow[i]);
        a.sum_r += g == 0 ? 1.0 : (double)l / (double)g;
        if (l > 0) {
            a.D += ((double)g / (double)l - 1.0) * s;
            a.num += s;
            a.den += s * ((double)g / (double)l);
        }
    }
    sh[threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        BatchStats t{0, 0, 0, 0};
        for (int i = 0; i < (int)blockDim.x; i++) {
            t.sum_r += sh[i].sum_r; t.D += sh[i].D; t.num += sh[i].num; t.den += sh[i].den;
        }
        *out = t;
    }
}

__global__ void k_sample_prep(const SampleParams* __restrict__ P, int32_t* __restrict__ seeds, int64_t* __restrict__ d_nt) {
    const int64_t n = P->n_batch;
    const int32_t* src = P->batch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        seeds[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_nt = n;
}

// seeds' epoch keys: h(seed, epoch, gid) = mix(seed ^ mix(epoch ^ mix(gid)))
__global__ void k_seed_keys(int64_t n, const int32_t* seeds, const int32_t* gid, uint64_t seed, uint64_t epoch,
                            uint64_t* keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = smix(seed ^ smix(epoch ^ smix((uint64_t)gid[seeds[i]])));
}

}  // namespace grappa

using namespace grappa;

struct BlockBufs {
    DevBuf rowptr, col, trowptr, tcol, inv_cnt, src, inv_cnt_node;
    int32_t n_dst = 0, n_src = 0;
    int64_t nnz = 0;
};

struct grappa_batch {
    int L = 0;
    int32_t n_batch = 0;
    BlockBufs blk[kMaxLayers];
    DevBuf picks, cnt, bitmap, where, erow, key_pad, skeys, svals, sort_tmp, counts, heavy_q;
    DevBuf scan_ws;                         // own scan partials (the sampler may run on a side stream)
    double c_uniform = 1, c_resampling = 1, c_hm = 1;
    // grappa_sample_async -> grappa_sample_wait: counts + stats land in pinned host memory
    void* host = nullptr;                   // int64 [3 kMaxLayers] + BatchStats
    cudaEvent_t done = nullptr;
    bool pending = false;
    // graph replay of the launch sequence (see grappa_sample_async): parameters in pinned host
    // memory (copied to `dparams` by the sequence), the seed copy, and the graph of the last key
    SampleParams* hparams = nullptr;
    DevBuf dparams, seedbuf;
    // graphs of the last few keys (the phases of an epoch cycle through the partitions), each valid
    // while none of the batch's buffers has moved since its capture (generation)
    struct Cached {
        std::vector<int64_t> key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        uint64_t gen = 0;
        uint64_t used = 0;
    };
    std::vector<Cached> graphs;
    std::vector<std::vector<int64_t>> seen;   // keys run eagerly once (capture on the next call)
    uint64_t gen = 0, tick = 0;
    int64_t nc_cap = 0;                        // node capacity of the buffers / launches
};
static constexpr int kSampleGraphs = 16;
// identity of every buffer the launch sequence touches: a change means a graph captured earlier
// points at freed memory
static uint64_t batch_layout(const grappa_batch* b) {
    uint64_t h = 1469598103934665603ull;
    auto mixp = [&](const void* p) { h = (h ^ (uint64_t)(uintptr_t)p) * 1099511628211ull; };
    for (int l = 0; l < kMaxLayers; l++)
        for (const DevBuf* d : {&b->blk[l].rowptr, &b->blk[l].col, &b->blk[l].trowptr, &b->blk[l].tcol,
                                &b->blk[l].inv_cnt, &b->blk[l].src, &b->blk[l].inv_cnt_node})
            mixp(d->p);
    for (const DevBuf* d : {&b->picks, &b->cnt, &b->bitmap, &b->where, &b->erow, &b->key_pad, &b->skeys,
                            &b->svals, &b->sort_tmp, &b->counts, &b->heavy_q, &b->scan_ws, &b->dparams, &b->seedbuf})
        mixp(d->p);
    return h;
}

static grappa_status sort_pairs(DevBuf& tmp, const int32_t* kin, int32_t* kout, const int32_t* vin,
                                int32_t* vout, int64_t n, int end_bit, cudaStream_t s) {
    GRAPPA_ARG(n < ((int64_t)1 << 31), GRAPPA_E_SUPPORT, "sampler: %lld items exceed cub's int sort limit",
               (long long)n);
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s);
    GRAPPA_TRY(tmp.grow(bytes));
    GRAPPA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s));
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_epoch_seeds(grappa_ctx* ctx, const grappa_part* part, uint64_t seed,
                                            int64_t epoch, int32_t* order, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && part && order, GRAPPA_E_ARG, "grappa_epoch_seeds: null argument");
    const grappa_part_info& I = part->info;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = I.n_seeds;
    // keys (uint64) + a stable radix sort of (key -> seed); input is ascending local id =
    // ascending global id, so equal keys keep gid order (R23 tie break)
    GRAPPA_TRY(ctx->red_ws.grow((size_t)n * 16 + 256));
    uint64_t* keys = (uint64_t*)ctx->red_ws.p;
    uint64_t* skeys = keys + n;
    k_seed_keys<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, s>>>(n, I.seeds, I.core_global, seed,
                                                                                      (uint64_t)epoch, keys);
    GRAPPA_LAUNCHED(ctx);
    GRAPPA_ARG(n < ((int64_t)1 << 31), GRAPPA_E_SUPPORT, "grappa_epoch_seeds: %lld seeds exceed the int sort limit",
               (long long)n);
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, skeys, I.seeds, order, (int)n, 0, 64, s);
    GRAPPA_TRY(ctx->scan_ws.grow(bytes));
    GRAPPA_CUDA(cub::DeviceRadixSort::SortPairs(ctx->scan_ws.p, bytes, keys, skeys, I.seeds, order, (int)n, 0, 64, s));
    ctx->launches++;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_sample(grappa_ctx* ctx, const grappa_part* part, const int32_t* batch,
                                       int32_t n_batch, const int32_t* fanouts, int32_t n_layers,
                                       uint64_t seed, int64_t epoch, int64_t batch_index,
                                       grappa_batch** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_TRY(grappa_sample_async(ctx, part, batch, n_batch, fanouts, n_layers, seed, epoch, batch_index,
                                   inout, stream));
    return grappa_sample_wait(*inout);
}

// The launch sequence of one batch: params H2D (pinned -> device), seed copy, per hop: frontier
// clear, Floyd pick (+ marking), unmark, two scans, block fill, radix-sort transpose, transpose
// rowptr; then the batch statistics.  Every size comes from device counters or from the call key
// (n_batch, fanouts, partition), so the sequence is the same for every batch of that key.
static grappa_status sample_body(grappa_ctx* ctx, grappa_batch* b, int64_t nc, int32_t n_batch,
                                 const int32_t* fanouts, int32_t n_layers, cudaStream_t s) {
    // nc: the node capacity the buffers and launches are sized for (>= the partition's n_core;
    // bitmap words past the partition stay zero, so scanning them adds nothing)
    int64_t* dc = (int64_t*)b->counts.p;
    BatchStats* dstat = (BatchStats*)(dc + 3 * kMaxLayers);
    SampleParams* dp = (SampleParams*)b->dparams.p;
    GRAPPA_CUDA(cudaMemcpyAsync(dp, b->hparams, sizeof(SampleParams), cudaMemcpyHostToDevice, s));
    k_sample_prep<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_batch, 256), 64)), 256, 0, s>>>(
        dp, (int32_t*)b->seedbuf.p, dc);
    GRAPPA_LAUNCHED(ctx);
    const int64_t nwords = ceil_div(nc, 32);
    int64_t cap_t = n_batch;
    const int32_t* targets = (const int32_t*)b->seedbuf.p;
    for (int h = 1; h <= n_layers; h++) {
        const int layer = n_layers - h;
        const int f = fanouts[layer];
        BlockBufs& B = b->blk[layer];
        int64_t* d_nt = dc + 3 * (h - 1);
        int64_t* d_ns = d_nt + 1;
        int64_t* d_nnz = d_nt + 2;
        const int64_t cap_s = std::min<int64_t>(nc, cap_t * (f + 1));
        const int64_t cap_nnz = cap_t * f;
        GRAPPA_TRY(b->picks.grow((size_t)cap_nnz * 4));
        GRAPPA_TRY(b->cnt.grow((size_t)cap_t * 4));
        GRAPPA_TRY(B.src.grow((size_t)cap_s * 4));
        GRAPPA_TRY(B.rowptr.grow((size_t)(cap_t + 1) * 8));
        GRAPPA_TRY(B.col.grow((size_t)cap_nnz * 4));
        GRAPPA_TRY(B.inv_cnt.grow((size_t)cap_t * 4));
        GRAPPA_TRY(B.inv_cnt_node.grow((size_t)cap_t * 4));
        GRAPPA_TRY(B.trowptr.grow((size_t)(cap_s + 1) * 8));
        GRAPPA_TRY(B.tcol.grow((size_t)cap_nnz * 4));
        GRAPPA_TRY(b->erow.grow((size_t)cap_nnz * 4));
        GRAPPA_TRY(b->key_pad.grow((size_t)cap_nnz * 4));
        GRAPPA_TRY(b->skeys.grow((size_t)cap_nnz * 4));
        const unsigned tgrid = (unsigned)std::min<int64_t>(ceil_div(cap_nnz, 256), (int64_t)ctx->sm_count * 16);
        GRAPPA_CUDA(cudaMemsetAsync(b->bitmap.p, 0, (size_t)nwords * 4, s));
        {
            auto kp = f <= 16 ? k_pick_floyd<16> : k_pick_floyd<32>;
            kp<<<(unsigned)std::min<int64_t>(ceil_div(cap_t, 256), (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
                d_nt, targets, dp, f, h - 1, (int32_t*)b->picks.p, (int32_t*)b->cnt.p, (uint32_t*)b->bitmap.p);
        }
        GRAPPA_LAUNCHED(ctx);
        k_unmark<<<(unsigned)std::min<int64_t>(ceil_div(cap_t, 256), 4096), 256, 0, s>>>(
            d_nt, targets, (uint32_t*)b->bitmap.p, (int32_t*)b->where.p, (int32_t*)B.src.p);
        GRAPPA_LAUNCHED(ctx);
        GRAPPA_TRY(device_scan(ctx, PopWord{(uint32_t*)b->bitmap.p}, nwords,
                               WriteNew{(uint32_t*)b->bitmap.p, d_nt, (int32_t*)B.src.p, (int32_t*)b->where.p, d_ns}, s,
                               nullptr, &b->scan_ws));
        GRAPPA_TRY(device_scan(ctx, CntUpTo{(int32_t*)b->cnt.p, d_nt}, cap_t,
                               WriteBRow{(int64_t*)B.rowptr.p, d_nnz}, s, nullptr, &b->scan_ws));
        (f <= 16 ? k_fill_block<16> : k_fill_block<32>)<<<tgrid, 256, 0, s>>>(d_nt, d_nnz, cap_nnz, (int32_t*)b->picks.p, (int32_t*)b->cnt.p, f,
                                           (int64_t*)B.rowptr.p, (int32_t*)b->where.p, (int32_t*)B.col.p,
                                           (int32_t*)b->erow.p, (int32_t*)b->key_pad.p, (float*)B.inv_cnt.p,
                                           targets, dp, (float*)B.inv_cnt_node.p);
        GRAPPA_LAUNCHED(ctx);
        int end_bit = 1;
        while (((int64_t)1 << end_bit) - 1 <= cap_s) end_bit++;
        GRAPPA_TRY(sort_pairs(b->sort_tmp, (int32_t*)b->key_pad.p, (int32_t*)b->skeys.p, (int32_t*)b->erow.p,
                              (int32_t*)B.tcol.p, cap_nnz, end_bit, s));
        ctx->launches++;
        k_trowptr<<<(unsigned)std::min<int64_t>(ceil_div(cap_nnz + 1, 256), 4096), 256, 0, s>>>(
            d_ns, d_nnz, (int32_t*)b->skeys.p, (int64_t*)B.trowptr.p);
        GRAPPA_LAUNCHED(ctx);
        // next hop: targets = this hop's sources
        if (h < n_layers) GRAPPA_CUDA(cudaMemcpyAsync(dc + 3 * h, d_ns, 8, cudaMemcpyDeviceToDevice, s));
        targets = (const int32_t*)B.src.p;
        cap_t = cap_s;
    }
    // batch coverage statistics over the seeds (hop 1 = output layer block)
    k_batch_stats<<<1, 256, 0, s>>>(n_batch, (const int32_t*)b->seedbuf.p, dp,
                                    (int64_t*)b->blk[n_layers - 1].rowptr.p, dstat);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

// Graph replay.  The ~45-launch sequence of a batch is launch-bound on the host (config 4 runs
// 2416 batches per epoch); since it only depends on the call key (partition arrays and sizes,
// n_batch, fanouts), the second call with a key captures it into a CUDA graph and later calls
// replay it (one graph launch; the parameters travel through the pinned `hparams`).  A call with
// another key runs eagerly and drops the graph (its buffers may move).  Results are the same
// launches on the same data whichever way they run.
extern "C" grappa_status grappa_sample_async(grappa_ctx* ctx, const grappa_part* part, const int32_t* batch,
                                             int32_t n_batch, const int32_t* fanouts, int32_t n_layers,
                                             uint64_t seed, int64_t epoch, int64_t batch_index,
                                             grappa_batch** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && part && batch && fanouts && inout, GRAPPA_E_ARG, "grappa_sample: null argument");
    GRAPPA_ARG(n_layers >= 1 && n_layers <= kMaxLayers, GRAPPA_E_ARG, "grappa_sample: 1 <= n_layers <= %d", kMaxLayers);
    GRAPPA_ARG(n_batch >= 1, GRAPPA_E_ARG, "grappa_sample: empty batch (S:213)");
    for (int l = 0; l < n_layers; l++)
        GRAPPA_ARG(fanouts[l] >= 1 && fanouts[l] <= kMaxFanout, GRAPPA_E_ARG,
                   "grappa_sample: fanout must be in [1, %d]", kMaxFanout);
    cudaStream_t s = (cudaStream_t)stream;
    const grappa_part_info& I = part->info;
    ProfScope ps(ctx, s, GRAPPA_K_SAMPLE, 0.0, 0.0);
    grappa_batch* b = *inout ? *inout : new grappa_batch();
    // the pinned parameters of the previous call on this batch object must have been consumed
    if (b->pending) {
        GRAPPA_CUDA(cudaEventSynchronize(b->done));
        b->pending = false;
    }
    b->L = n_layers;
    b->n_batch = n_batch;
    // node capacity of the launch sequence: grows with 1/8 headroom, so one recorded sequence
    // serves every partition of a run (their sizes differ by a few %)
    if (I.n_core > b->nc_cap) b->nc_cap = I.n_core + I.n_core / 8;
    const int64_t nc = b->nc_cap;
    // device counters: per hop n_t, n_s, nnz (3 x kMaxLayers int64) + stats
    GRAPPA_TRY(b->counts.grow(3 * kMaxLayers * 8 + sizeof(BatchStats) + 64));
    GRAPPA_TRY(b->bitmap.grow((size_t)ceil_div(nc, 32) * 4));
    GRAPPA_TRY(b->where.grow((size_t)nc * 4));
    GRAPPA_TRY(b->dparams.grow(sizeof(SampleParams)));
    GRAPPA_TRY(b->seedbuf.grow((size_t)n_batch * 4));
    if (!b->hparams) GRAPPA_CUDA(cudaMallocHost((void**)&b->hparams, sizeof(SampleParams)));
    if (!b->host) {
        GRAPPA_CUDA(cudaMallocHost(&b->host, sizeof(int64_t) * 3 * kMaxLayers + sizeof(BatchStats)));
        GRAPPA_CUDA(cudaEventCreateWithFlags(&b->done, cudaEventDisableTiming));
    }
    SampleParams& P = *b->hparams;
    P.n_batch = n_batch;
    P.batch = batch;
    P.rowptr = I.rowptr;
    P.col = I.col;
    P.gid = I.core_global;
    P.d_l = I.d_l;
    P.d_g = I.d_g;
    for (int h = 1; h <= n_layers; h++)
        // h(seed, epoch, batch, hop) = mix(seed ^ mix(epoch ^ mix(batch ^ mix(hop))))
        P.key[h - 1] = hmix(seed ^ hmix((uint64_t)epoch ^ hmix((uint64_t)batch_index ^ hmix((uint64_t)h))));
    // every size the sequence is launched with (the partition itself is a parameter)
    std::vector<int64_t> key = {nc, n_batch, n_layers};
    for (int l = 0; l < n_layers; l++) key.push_back(fanouts[l]);
    // not on the legacy default stream (cannot be captured), not inside a caller's own capture,
    // not while per-kernel-class profiling records events
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    const bool can_graph = !ctx->profiling && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread &&
                           cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusNone;
    const uint64_t layout = batch_layout(b);
    if (layout != b->gen) {                   // buffers moved: every cached graph is stale
        for (auto& c : b->graphs) cudaGraphExecDestroy(c.exec);
        b->graphs.clear();
        b->gen = layout;
    }
    b->tick++;
    grappa_batch::Cached* hit = nullptr;
    for (auto& c : b->graphs)
        if (c.key == key) hit = &c;
    bool seen = false;
    for (auto& k : b->seen)
        if (k == key) seen = true;
    if (can_graph && hit) {
        hit->used = b->tick;
        GRAPPA_CUDA(cudaGraphLaunch(hit->exec, s));
        ctx->launches += hit->launches;
    } else if (can_graph && seen) {
        // capture the sequence (buffers already sized by the eager call with this key)
        const int64_t l0 = ctx->launches;
        GRAPPA_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const grappa_status st = sample_body(ctx, b, nc, n_batch, fanouts, n_layers, s);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        grappa_batch::Cached c;
        cudaError_t ie = cudaErrorUnknown;
        if (st == GRAPPA_OK && ce == cudaSuccess && batch_layout(b) == b->gen) ie = cudaGraphInstantiate(&c.exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
            // the sequence could not be captured as it stands (e.g. a buffer had to grow inside
            // the capture): run it eagerly; the next call with this key tries again
            cudaGetLastError();
            ctx->launches = l0;
            GRAPPA_TRY(sample_body(ctx, b, nc, n_batch, fanouts, n_layers, s));
            b->gen = batch_layout(b);
            for (auto& x : b->graphs) cudaGraphExecDestroy(x.exec);
            b->graphs.clear();
            goto published;
        }
        c.key = key;
        c.launches = ctx->launches - l0;
        c.gen = b->gen;
        c.used = b->tick;
        if ((int)b->graphs.size() >= kSampleGraphs) {     // drop the least recently used
            size_t lru = 0;
            for (size_t i = 1; i < b->graphs.size(); i++)
                if (b->graphs[i].used < b->graphs[lru].used) lru = i;
            cudaGraphExecDestroy(b->graphs[lru].exec);
            b->graphs.erase(b->graphs.begin() + lru);
        }
        b->graphs.push_back(c);
        GRAPPA_CUDA(cudaGraphLaunch(c.exec, s));
    } else {
        GRAPPA_TRY(sample_body(ctx, b, nc, n_batch, fanouts, n_layers, s));
        if (batch_layout(b) != b->gen) {             // this call moved buffers
            for (auto& c : b->graphs) cudaGraphExecDestroy(c.exec);
            b->graphs.clear();
            b->gen = batch_layout(b);
        }
        if (!seen) {
            b->seen.push_back(key);
            if ((int)b->seen.size() > 4 * kSampleGraphs) b->seen.erase(b->seen.begin());
        }
    }
published:
    GRAPPA_CUDA(cudaMemcpyAsync(b->host, b->counts.p, sizeof(int64_t) * 3 * kMaxLayers + sizeof(BatchStats),
                                cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaEventRecord(b->done, s));
    b->pending = true;
    *inout = b;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_sample_event(const grappa_batch* b, void** event_out) {
    GRAPPA_ARG(b && event_out, GRAPPA_E_ARG, "grappa_sample_event: null argument");
    *event_out = (void*)b->done;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_sample_wait(grappa_batch* b) {
    GRAPPA_ARG(b, GRAPPA_E_ARG, "grappa_sample_wait: null argument");
    if (!b->pending) return GRAPPA_OK;
    GRAPPA_CUDA(cudaEventSynchronize(b->done));
    b->pending = false;
    const int n_layers = b->L, n_batch = b->n_batch;
    const int64_t* hc = (const int64_t*)b->host;
    BatchStats hs;
    memcpy(&hs, hc + 3 * kMaxLayers, sizeof(hs));
    for (int h = 1; h <= n_layers; h++) {
        BlockBufs& B = b->blk[n_layers - h];
        B.n_dst = (int32_t)hc[3 * (h - 1)];
        B.n_src = (int32_t)hc[3 * (h - 1) + 1];
        B.nnz = hc[3 * (h - 1) + 2];
    }
    b->c_uniform = hs.sum_r / (double)n_batch;
    b->c_resampling = hs.D < 1e-9 ? 1.0 : std::min(1.0 / hs.D, 10.0);
    b->c_hm = hs.num > 0 ? hs.num / hs.den : 1.0;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_batch_query(const grappa_batch* b, int32_t layer, grappa_block_info* out) {
    GRAPPA_ARG(b && out, GRAPPA_E_ARG, "grappa_batch_query: null argument");
    GRAPPA_ARG(layer >= 0 && layer < b->L, GRAPPA_E_ARG, "grappa_batch_query: layer out of range");
    GRAPPA_ARG(!b->pending, GRAPPA_E_ARG, "grappa_batch_query: batch not published (grappa_sample_wait)");
    const BlockBufs& B = b->blk[layer];
    out->n_dst = B.n_dst; out->n_src = B.n_src; out->nnz = B.nnz;
    out->rowptr = (const int64_t*)B.rowptr.p; out->col = (const int32_t*)B.col.p;
    out->t_rowptr = (const int64_t*)B.trowptr.p; out->t_col = (const int32_t*)B.tcol.p;
    out->inv_cnt = (const float*)B.inv_cnt.p; out->src = (const int32_t*)B.src.p;
    out->inv_cnt_node = (const float*)B.inv_cnt_node.p;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_batch_factors(const grappa_batch* b, double* cu, double* cr, double* ch) {
    GRAPPA_ARG(b && cu && cr && ch, GRAPPA_E_ARG, "grappa_batch_factors: null argument");
    GRAPPA_ARG(!b->pending, GRAPPA_E_ARG, "grappa_batch_factors: batch not published (grappa_sample_wait)");
    *cu = b->c_uniform; *cr = b->c_resampling; *ch = b->c_hm;
    return GRAPPA_OK;
}

extern "C" void grappa_batch_destroy(grappa_batch* b) {
    if (!b) return;
    if (b->done) { cudaEventSynchronize(b->done); cudaEventDestroy(b->done); }
    if (b->host) cudaFreeHost(b->host);
    if (b->hparams) cudaFreeHost(b->hparams);
    for (auto& c : b->graphs) cudaGraphExecDestroy(c.exec);
    b->dparams.release();
    b->seedbuf.release();
    for (int l = 0; l < kMaxLayers; l++)
        for (DevBuf* d : {&b->blk[l].rowptr, &b->blk[l].col, &b->blk[l].trowptr, &b->blk[l].tcol,
                          &b->blk[l].inv_cnt, &b->blk[l].src, &b->blk[l].inv_cnt_node})
            d->release();
    for (DevBuf* d : {&b->picks, &b->cnt, &b->bitmap, &b->where, &b->erow, &b->key_pad, &b->skeys,
                      &b->svals, &b->sort_tmp, &b->counts, &b->heavy_q, &b->scan_ws})
        d->release();
    delete b;
}

// ------------------------------------------------------------------------------ step
namespace {
struct StepLayout {
    size_t H[kMaxLayers + 1], M[kMaxLayers], dz[2], dM, splitk, total;
};
StepLayout step_layout(const grappa_batch* b, int L, const int32_t* dp, grappa_dtype dt) {
    const size_t es = dt == GRAPPA_BF16 ? 2 : 4;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    StepLayout s{};
    size_t off = 0;
    s.H[0] = off; off += al((size_t)b->blk[0].n_src * dp[0] * es);
    size_t dz_max = 0, dm_max = 0, sk_max = 0;
    for (int l = 0; l < L; l++) {
        const BlockBufs& B = b->blk[l];
        s.H[l + 1] = off; off += al((size_t)B.n_dst * dp[l + 1] * es);
        s.M[l] = off; off += al((size_t)B.n_dst * dp[l] * es);
        dz_max = std::max(dz_max, (size_t)B.n_src * dp[l] * es);
        dz_max = std::max(dz_max, (size_t)B.n_dst * dp[l + 1] * es);
        dm_max = std::max(dm_max, (size_t)B.n_dst * dp[l] * es);
        sk_max = std::max(sk_max, gemm_tn_ws_bytes(B.n_dst, dp[l], dp[l], dp[l + 1]));
    }
    s.dz[0] = off; off += al(dz_max);
    s.dz[1] = off; off += al(dz_max);
    s.dM = off; off += al(dm_max);
    s.splitk = off; off += al(sk_max);
    s.total = off;
    return s;
}
}  // namespace

extern "C" size_t grappa_minibatch_ws_bytes(const grappa_batch* b, int32_t L, const int32_t* dims_pad,
                                            grappa_dtype dtype) {
    if (!b || !dims_pad || L != b->L || b->pending) return 0;
    return step_layout(b, L, dims_pad, dtype).total;
}

extern "C" grappa_status grappa_minibatch_step(grappa_ctx* ctx, const grappa_part* part, const grappa_batch* b,
                                               int32_t L, const int32_t* dp, int32_t num_classes,
                                               const float* theta, float* grad, void* ws, size_t ws_bytes,
                                               double* loss_dev, void* const* hidden_out, grappa_dtype dt,
                                               void* stream) {
    CallScope call_scope(ctx, stream);
    return grappa_minibatch_step_ex(ctx, part, b, L, dp, num_classes, theta, grad, ws, ws_bytes, loss_dev,
                                    hidden_out, dt, 0u, stream);
}

extern "C" grappa_status grappa_minibatch_step_ex(grappa_ctx* ctx, const grappa_part* part, const grappa_batch* b,
                                                  int32_t L, const int32_t* dp, int32_t num_classes,
                                                  const float* theta, float* grad, void* ws, size_t ws_bytes,
                                                  double* loss_dev, void* const* hidden_out, grappa_dtype dt,
                                                  unsigned flags, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG((flags & ~GRAPPA_LAYER_NODE_LEVEL) == 0, GRAPPA_E_ARG,
               "grappa_minibatch_step_ex: flags 0x%x invalid", flags);
    const bool node = flags & GRAPPA_LAYER_NODE_LEVEL;
    GRAPPA_ARG(ctx && part && b && dp && theta && grad && ws && loss_dev, GRAPPA_E_ARG,
               "grappa_minibatch_step: null argument");
    GRAPPA_ARG(L == b->L, GRAPPA_E_ARG, "grappa_minibatch_step: n_layers %d != sampled %d", L, b->L);
    GRAPPA_ARG(!b->pending, GRAPPA_E_ARG, "grappa_minibatch_step: batch not published (grappa_sample_wait)");
    // the blocks may have been sampled on another stream (grappa_sample_async): order after them
    if (b->done) GRAPPA_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, b->done, 0));
    for (int l = 0; l <= L; l++)
        GRAPPA_ARG(dp[l] > 0 && dp[l] % 16 == 0, GRAPPA_E_SHAPE, "grappa_minibatch_step: dims must be multiples of 16");
    GRAPPA_ARG(dp[0] == part->info.feat_dim && dt == part->info.dtype, GRAPPA_E_SHAPE,
               "grappa_minibatch_step: dims_pad[0]/dtype must match the partition features");
    GRAPPA_ARG(num_classes >= 1 && num_classes <= dp[L], GRAPPA_E_ARG, "grappa_minibatch_step: bad num_classes");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = dt == GRAPPA_BF16 ? 2 : 4;
    const StepLayout lay = step_layout(b, L, dp, dt);
    GRAPPA_ARG(ws_bytes >= lay.total, GRAPPA_E_ARG,
               "grappa_minibatch_step: workspace %zu B < %zu B needed by this batch", ws_bytes, lay.total);
    char* w = (char*)ws;
    // h_0 = features of the outermost sources
    const BlockBufs& B0 = b->blk[0];
    k_gather_rows<<<(unsigned)std::min<int64_t>(ceil_div(B0.n_src, 8), (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
        B0.n_src, (int64_t)dp[0] * es, (const int32_t*)B0.src.p, (const uint4*)part->info.x, (uint4*)(w + lay.H[0]));
    GRAPPA_LAUNCHED(ctx);
    std::vector<size_t> woff(L + 1, 0);
    for (int l = 0; l < L; l++) woff[l + 1] = woff[l] + (size_t)2 * dp[l] * dp[l + 1];
    for (int l = 0; l < L; l++) {
        const BlockBufs& B = b->blk[l];
        SpmmArgs a;
        a.n = B.n_dst; a.nnz = B.nnz; a.rowptr = (const int64_t*)B.rowptr.p; a.col = (const int32_t*)B.col.p;
        a.X = w + lay.H[l]; a.width = dp[l];
        a.row_scale = (const float*)(node ? B.inv_cnt_node.p : B.inv_cnt.p); a.out = w + lay.M[l];
        GRAPPA_TRY(spmm_csr(ctx, a, dt, s));
        GemmArgs g;
        g.M = B.n_dst; g.K1 = dp[l]; g.K2 = dp[l]; g.N = dp[l + 1];
        g.A1 = w + lay.H[l]; g.A2 = w + lay.M[l]; g.B = theta + woff[l];
        g.relu = l < L - 1; g.n_split = dp[l + 1]; g.C1 = w + lay.H[l + 1];
        GRAPPA_TRY(gemm_nn(ctx, g, dt, s));
        if (hidden_out && l < L - 1 && hidden_out[l])
            GRAPPA_CUDA(cudaMemcpyAsync(hidden_out[l], w + lay.H[l + 1], (size_t)B.n_dst * dp[l + 1] * es,
                                        cudaMemcpyDeviceToDevice, s));
    }
    // loss over the batch seeds = the first n_batch rows of the output layer
    const BlockBufs& BL = b->blk[L - 1];
    char* dz = w + lay.dz[0];
    GRAPPA_TRY(loss_rows(ctx, b->n_batch, nullptr, (const int32_t*)BL.src.p, part->info.labels, BL.n_dst,
                         w + lay.H[L], num_classes, dp[L], dz, loss_dev, dt, s));
    int cur = 0;
    for (int l = L - 1; l >= 0; l--) {
        const BlockBufs& B = b->blk[l];
        GemmTNArgs t;
        t.M = B.n_dst; t.K1 = dp[l]; t.K2 = dp[l]; t.N = dp[l + 1];
        t.A1 = w + lay.H[l]; t.A2 = w + lay.M[l]; t.B = dz; t.C = grad + woff[l]; t.ws = (float*)(w + lay.splitk);
        GRAPPA_TRY(gemm_tn(ctx, t, dt, s));
        if (l == 0) break;
        char* dz_in = w + lay.dz[cur ^ 1];
        GemmArgs g;
        g.M = B.n_dst; g.K1 = dp[l + 1]; g.N = 2 * dp[l]; g.A1 = dz; g.B = theta + woff[l]; g.b_trans = 1;
        g.n_split = dp[l]; g.C1 = dz_in; g.C2 = w + lay.dM;
        GRAPPA_TRY(gemm_nn(ctx, g, dt, s));
        // source-only rows (n_dst .. n_src) have no dh_s term: the SpMM writes them instead of
        // accumulating (no zero fill of dz_in's tail)
        SpmmArgs a;
        a.n = B.n_src; a.nnz = B.nnz; a.rowptr = (const int64_t*)B.trowptr.p; a.col = (const int32_t*)B.tcol.p;
        a.X = w + lay.dM; a.width = dp[l];
        a.col_scale = (const float*)(node ? B.inv_cnt_node.p : B.inv_cnt.p); a.accumulate = 1;
        a.acc_rows = B.n_dst;
        a.mask = w + lay.H[l]; a.out = dz_in;
        GRAPPA_TRY(spmm_csr(ctx, a, dt, s));
        dz = dz_in;
        cur ^= 1;
    }
    return GRAPPA_OK;
}
