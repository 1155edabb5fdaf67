// shard.cu -- sharded mode of a3: chunk shards, their NCCL exchange at a super-epoch switch,
// and the merge of two shards into the source CSR the repartition pipeline consumes.
//
// PAPER: P:198 (§3.3 chunks stored once, a partition = base chunk + swept chunk), P:413 (§4 "at
// a switch, workers load the new chunk's edges"), P:416 (data moves only at switches; the
// per-iteration traffic is the gradient all-reduce).  SURVEY §8(a) a3 (i), §8(e).
//
// A shard is one chunk's rows: node ids ascending, their full adjacency (global ids, sorted),
// features, labels, train flags.  With W = C and G ranks, rank r owns the chunks c = r mod G;
// at super-epoch t worker w needs the swept chunk (w + t) mod C from its owner -- a shift
// permutation of point-to-point transfers (engine.shard_plan).  Everything here is integer
// index work or byte copies, so the partition built from two shards is bitwise the one the
// replicated path builds (tests/test_gpu_shard.py).
#include <nccl.h>

#include <string>
#include "part.cuh"
#include "scan.cuh"

#include <vector>

namespace grappa {

struct ShFlagChunk {
    const int32_t* chunk_of; int32_t c;
    __device__ int32_t operator()(int64_t v) const { return chunk_of[v] == c; }
};
struct ShWriteIds {
    int32_t* ids; int64_t* stat;
    __device__ void operator()(int64_t v, int64_t p, int32_t f) const {
        if (f) ids[p] = (int32_t)v;
    }
    __device__ void finish(int64_t, int64_t total) const { stat[0] = total; }
};
struct ShReadDeg {
    const int32_t* ids; const int64_t* g_rowptr;
    __device__ int32_t operator()(int64_t j) const {
        const int32_t v = ids[j];
        return (int32_t)(g_rowptr[v + 1] - g_rowptr[v]);
    }
};
struct ShReadI32 {
    const int32_t* a;
    __device__ int32_t operator()(int64_t i) const { return a[i]; }
};
struct ShWriteRowptr {
    int64_t* rowptr; int64_t* stat;
    __device__ void operator()(int64_t i, int64_t p, int32_t) const { rowptr[i] = p; }
    __device__ void finish(int64_t n, int64_t total) const { rowptr[n] = total; stat[1] = total; }
};

// warp per shard row: copy the global row, label and train flag
__global__ void k_shard_rows(int64_t n_rows, const int32_t* __restrict__ ids, const int64_t* __restrict__ g_rowptr,
                             const int32_t* __restrict__ g_col, const int32_t* __restrict__ g_labels,
                             const uint8_t* __restrict__ g_train, const int64_t* __restrict__ rowptr,
                             int32_t* __restrict__ col, int32_t* __restrict__ labels, uint8_t* __restrict__ train) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_rows; j += nw) {
        const int32_t v = ids[j];
        const int64_t a = g_rowptr[v], d = g_rowptr[v + 1] - a, o = rowptr[j];
        for (int64_t e = lane; e < d; e += 32) col[o + e] = g_col[a + e];
        if (lane == 0) {
            labels[j] = g_labels ? g_labels[v] : 0;
            train[j] = g_train[v];
        }
    }
}

// shard row j -> its local id rank[ids[j]] in the chunk pair: source code (shard << 32 | j), degree
__global__ void k_shard_place(int64_t n_rows, int64_t tag, const int32_t* __restrict__ ids,
                              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ rank,
                              int64_t* __restrict__ m_src, int32_t* __restrict__ m_deg) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_rows;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = rank[ids[j]];
        m_src[i] = (tag << 32) | j;
        m_deg[i] = (int32_t)(rowptr[j + 1] - rowptr[j]);
    }
}

struct ShardView {
    const int64_t* rowptr; const int32_t* col; const uint4* x; const int32_t* labels; const uint8_t* train;
};

// warp per local row: copy its shard row (adjacency, feature row, label, train flag)
__global__ void k_shard_merge(int64_t n_core, ShardView A, ShardView B, const int64_t* __restrict__ m_src,
                              const int64_t* __restrict__ m_rowptr, int32_t* __restrict__ m_col,
                              int32_t* __restrict__ m_lab, uint8_t* __restrict__ m_tr, uint4* __restrict__ x_out,
                              int64_t vec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_core; i += nw) {
        const int64_t code = m_src[i];
        const ShardView& S = (code >> 32) ? B : A;
        const int64_t j = code & 0xffffffffll;
        const int64_t a = S.rowptr[j], d = S.rowptr[j + 1] - a, o = m_rowptr[i];
        for (int64_t e = lane; e < d; e += 32) m_col[o + e] = S.col[a + e];
        if (x_out)
            for (int64_t k = lane; k < vec; k += 32) x_out[i * vec + k] = S.x[j * vec + k];
        if (lane == 0) {
            m_lab[i] = S.labels[j];
            m_tr[i] = S.train[j];
        }
    }
}

static unsigned sh_grid(grappa_ctx* ctx, int64_t items, int per_block) {
    int64_t b = ceil_div(items > 0 ? items : 1, per_block);
    int64_t cap = (int64_t)ctx->sm_count * 16;
    return (unsigned)(b > cap ? cap : b);
}

grappa_status shard_merge(grappa_ctx* ctx, const grappa_shard* sa, const grappa_shard* sb, const int32_t* rank,
                          int64_t n_core, int64_t* m_src, int32_t* m_deg, int64_t* m_rowptr, int32_t* m_col,
                          int32_t* m_lab, uint8_t* m_tr, void* x_out, int64_t row_bytes, int64_t* d_stat,
                          cudaStream_t s) {
    const grappa_shard_info &A = sa->info, &B = sb->info;
    GRAPPA_ARG(A.n_rows + B.n_rows == n_core, GRAPPA_E_ARG,
               "grappa_repartition_shards: shard rows (%lld + %lld) do not match the chunk map (%lld core nodes)",
               (long long)A.n_rows, (long long)B.n_rows, (long long)n_core);
    k_shard_place<<<sh_grid(ctx, A.n_rows, 256), 256, 0, s>>>(A.n_rows, 0, A.ids, A.rowptr, rank, m_src, m_deg);
    GRAPPA_LAUNCHED(ctx);
    k_shard_place<<<sh_grid(ctx, B.n_rows, 256), 256, 0, s>>>(B.n_rows, 1, B.ids, B.rowptr, rank, m_src, m_deg);
    GRAPPA_LAUNCHED(ctx);
    GRAPPA_TRY(device_scan(ctx, ShReadI32{m_deg}, n_core, ShWriteRowptr{m_rowptr, d_stat + 6}, s));
    ShardView va{A.rowptr, A.col, (const uint4*)A.x, A.labels, A.train};
    ShardView vb{B.rowptr, B.col, (const uint4*)B.x, B.labels, B.train};
    k_shard_merge<<<sh_grid(ctx, n_core, 8), 256, 0, s>>>(n_core, va, vb, m_src, m_rowptr, m_col, m_lab, m_tr,
                                                          (uint4*)x_out, row_bytes / 16);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

static void shard_publish(grappa_shard* sh, int32_t chunk, int64_t n_rows, int64_t nnz, int32_t feat_dim,
                          grappa_dtype dtype) {
    grappa_shard_info& I = sh->info;
    I.chunk = chunk; I.n_rows = n_rows; I.nnz = nnz; I.feat_dim = feat_dim; I.dtype = dtype;
    I.ids = (const int32_t*)sh->ids.p; I.rowptr = (const int64_t*)sh->rowptr.p; I.col = (const int32_t*)sh->col.p;
    I.x = feat_dim ? sh->x.p : nullptr; I.labels = (const int32_t*)sh->labels.p;
    I.train = (const uint8_t*)sh->train.p;
}

static grappa_status shard_alloc(grappa_shard* sh, int64_t n_rows, int64_t nnz, int32_t feat_dim, grappa_dtype dtype) {
    const int64_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
    GRAPPA_TRY(sh->ids.grow((size_t)(n_rows > 0 ? n_rows : 1) * 4));
    GRAPPA_TRY(sh->rowptr.grow((size_t)(n_rows + 1) * 8));
    GRAPPA_TRY(sh->col.grow((size_t)(nnz > 0 ? nnz : 1) * 4));
    GRAPPA_TRY(sh->labels.grow((size_t)(n_rows > 0 ? n_rows : 1) * 4));
    GRAPPA_TRY(sh->train.grow((size_t)(n_rows > 0 ? n_rows : 1)));
    if (feat_dim) GRAPPA_TRY(sh->x.grow((size_t)(n_rows > 0 ? n_rows : 1) * feat_dim * esz));
    return GRAPPA_OK;
}

}  // namespace grappa

using namespace grappa;

extern "C" grappa_status grappa_shard_extract(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                              int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                              int32_t num_chunks, int32_t chunk, const uint8_t* train_mask,
                                              const int32_t* labels, grappa_shard** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && g && chunk_of && train_mask && inout, GRAPPA_E_ARG, "grappa_shard_extract: null argument");
    GRAPPA_ARG(chunk >= 0 && chunk < num_chunks, GRAPPA_E_ARG, "grappa_shard_extract: chunk %d out of range", chunk);
    GRAPPA_ARG(feats == nullptr || (feat_dim > 0 && feat_dim % 16 == 0), GRAPPA_E_SHAPE,
               "grappa_shard_extract: feat_dim must be a positive multiple of 16");
    GRAPPA_ARG(g->num_nodes > 0 && g->num_nodes < (1ll << 31), GRAPPA_E_ARG,
               "grappa_shard_extract: num_nodes out of int32 range");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = g->num_nodes;
    grappa_shard* sh = *inout ? *inout : new grappa_shard();
    auto fail = [&](grappa_status st) {
        if (!*inout) grappa_shard_destroy(sh);
        return st;
    };
#define SH_TRY(expr)                          \
    do {                                      \
        grappa_status _s = (expr);            \
        if (_s != GRAPPA_OK) return fail(_s); \
    } while (0)
    SH_TRY(ctx->small.grow(16 * sizeof(int64_t)));
    int64_t* d_stat = (int64_t*)ctx->small.p;
    // ids compacted into the ctx's N-sized workspace, then copied into the shard at its size
    SH_TRY(ctx->red_ws.grow((size_t)N * 4));
    SH_TRY(device_scan(ctx, ShFlagChunk{chunk_of, chunk}, N, ShWriteIds{(int32_t*)ctx->red_ws.p, d_stat}, s));
    int64_t n_rows = 0;
    if (cudaMemcpyAsync(&n_rows, d_stat, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("grappa_shard_extract: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    GRAPPA_ARG(n_rows > 0, fail(GRAPPA_E_EMPTY), "grappa_shard_extract: chunk %d is empty", chunk);
    SH_TRY(sh->ids.grow((size_t)n_rows * 4));
    if (cudaMemcpyAsync(sh->ids.p, ctx->red_ws.p, (size_t)n_rows * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
        set_error("grappa_shard_extract: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    SH_TRY(sh->rowptr.grow((size_t)(n_rows + 1) * 8));
    SH_TRY(device_scan(ctx, ShReadDeg{(const int32_t*)sh->ids.p, g->rowptr}, n_rows,
                       ShWriteRowptr{(int64_t*)sh->rowptr.p, d_stat}, s));
    int64_t nnz = 0;
    if (cudaMemcpyAsync(&nnz, d_stat + 1, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("grappa_shard_extract: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(GRAPPA_E_CUDA);
    }
    const int32_t fd = feats ? feat_dim : 0;
    SH_TRY(shard_alloc(sh, n_rows, nnz, fd, dtype));
    k_shard_rows<<<sh_grid(ctx, n_rows, 8), 256, 0, s>>>(n_rows, (const int32_t*)sh->ids.p, g->rowptr, g->col,
                                                         labels, train_mask, (const int64_t*)sh->rowptr.p,
                                                         (int32_t*)sh->col.p, (int32_t*)sh->labels.p,
                                                         (uint8_t*)sh->train.p);
    GRAPPA_LAUNCHED(ctx);
    if (fd) {
        const int64_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
        k_gather_rows<<<sh_grid(ctx, n_rows, 8), 256, 0, s>>>(n_rows, fd * esz, (const int32_t*)sh->ids.p,
                                                              (const uint4*)feats, (uint4*)sh->x.p);
        GRAPPA_LAUNCHED(ctx);
    }
    shard_publish(sh, chunk, n_rows, nnz, fd, dtype);
    *inout = sh;
    return GRAPPA_OK;
#undef SH_TRY
}

extern "C" grappa_status grappa_shard_query(const grappa_shard* shard, grappa_shard_info* out) {
    GRAPPA_ARG(shard && out, GRAPPA_E_ARG, "grappa_shard_query: null argument");
    *out = shard->info;
    return GRAPPA_OK;
}

extern "C" void grappa_shard_destroy(grappa_shard* sh) {
    if (!sh) return;
    sh->ids.release();
    sh->rowptr.release();
    sh->col.release();
    sh->x.release();
    sh->labels.release();
    sh->train.release();
    delete sh;
}

#define SH_NCCL(expr)                                                                     \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess) {                                                          \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(_r)); \
            return GRAPPA_E_NCCL;                                                         \
        }                                                                                 \
    } while (0)

extern "C" grappa_status grappa_shard_exchange(grappa_ctx* ctx, int32_t n_xfers, const grappa_shard_xfer* xfers,
                                               void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && (n_xfers == 0 || xfers) && n_xfers >= 0, GRAPPA_E_ARG, "grappa_shard_exchange: null argument");
    GRAPPA_ARG(ctx->comm, GRAPPA_E_ARG, "grappa_shard_exchange: the ctx has no NCCL communicator");
    for (int32_t k = 0; k < n_xfers; k++) {
        const grappa_shard_xfer& x = xfers[k];
        GRAPPA_ARG(x.peer >= 0 && x.peer < ctx->nranks, GRAPPA_E_ARG, "grappa_shard_exchange: bad peer %d", x.peer);
        GRAPPA_ARG((x.send != nullptr) != (x.recv != nullptr), GRAPPA_E_ARG,
                   "grappa_shard_exchange: transfer %d must either send or receive", k);
    }
    if (n_xfers == 0) return GRAPPA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    ncclComm_t comm = (ncclComm_t)ctx->comm;
    // round 1: headers {chunk, n_rows, nnz, feat_dim | dtype << 32}
    std::vector<int64_t> hdr((size_t)n_xfers * 4, 0);
    for (int32_t k = 0; k < n_xfers; k++)
        if (xfers[k].send) {
            const grappa_shard_info& I = xfers[k].send->info;
            hdr[k * 4 + 0] = I.chunk;
            hdr[k * 4 + 1] = I.n_rows;
            hdr[k * 4 + 2] = I.nnz;
            hdr[k * 4 + 3] = (int64_t)I.feat_dim | ((int64_t)I.dtype << 32);
        }
    GRAPPA_TRY(ctx->xf_hdr.grow((size_t)n_xfers * 40));
    int64_t* d_hdr = (int64_t*)ctx->xf_hdr.p;
    GRAPPA_CUDA(cudaMemcpyAsync(d_hdr, hdr.data(), (size_t)n_xfers * 32, cudaMemcpyHostToDevice, s));
    SH_NCCL(ncclGroupStart());
    for (int32_t k = 0; k < n_xfers; k++) {
        if (xfers[k].send) SH_NCCL(ncclSend(d_hdr + k * 4, 4, ncclInt64, xfers[k].peer, comm, s));
        else SH_NCCL(ncclRecv(d_hdr + k * 4, 4, ncclInt64, xfers[k].peer, comm, s));
    }
    SH_NCCL(ncclGroupEnd());
    GRAPPA_CUDA(cudaMemcpyAsync(hdr.data(), d_hdr, (size_t)n_xfers * 32, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    // size the receive shards; a receiver that cannot take a shard does not return yet: both sides
    // of every transfer first agree on success (round 1b), so no sender is left in round 2 with a
    // ncclSend nobody matches
    std::vector<grappa_shard*> rs((size_t)n_xfers, nullptr);
    std::vector<int64_t> ok((size_t)n_xfers, 0);
    grappa_status local = GRAPPA_OK;
    std::string local_msg;
    for (int32_t k = 0; k < n_xfers; k++) {
        if (!xfers[k].recv) continue;
        const int64_t n_rows = hdr[k * 4 + 1], nnz = hdr[k * 4 + 2];
        const int32_t fd = (int32_t)(hdr[k * 4 + 3] & 0xffffffffll);
        const grappa_dtype dt = (grappa_dtype)(hdr[k * 4 + 3] >> 32);
        grappa_status st = GRAPPA_OK;
        if (local != GRAPPA_OK) {
            st = local;
        } else if (!(n_rows > 0 && nnz >= 0 && fd >= 0 && (dt == GRAPPA_F32 || dt == GRAPPA_BF16))) {
            set_error("grappa_shard_exchange: malformed header from rank %d", xfers[k].peer);
            st = GRAPPA_E_ARG;
        } else {
            grappa_shard* sh = *xfers[k].recv ? *xfers[k].recv : new grappa_shard();
            st = shard_alloc(sh, n_rows, nnz, fd, dt);
            if (st != GRAPPA_OK) {
                if (!*xfers[k].recv) grappa_shard_destroy(sh);
            } else {
                shard_publish(sh, (int32_t)hdr[k * 4 + 0], n_rows, nnz, fd, dt);
                *xfers[k].recv = sh;
                rs[k] = sh;
            }
        }
        if (st != GRAPPA_OK && local == GRAPPA_OK) {
            local = st;
            local_msg = grappa_last_error();
        }
        ok[k] = st == GRAPPA_OK ? 1 : 0;
    }
    // round 1b: every receiver tells its sender whether it can take the arrays
    int64_t* d_ok = d_hdr + (size_t)n_xfers * 4;
    GRAPPA_CUDA(cudaMemcpyAsync(d_ok, ok.data(), (size_t)n_xfers * 8, cudaMemcpyHostToDevice, s));
    SH_NCCL(ncclGroupStart());
    for (int32_t k = 0; k < n_xfers; k++) {
        if (xfers[k].recv) SH_NCCL(ncclSend(d_ok + k, 1, ncclInt64, xfers[k].peer, comm, s));
        else SH_NCCL(ncclRecv(d_ok + k, 1, ncclInt64, xfers[k].peer, comm, s));
    }
    SH_NCCL(ncclGroupEnd());
    GRAPPA_CUDA(cudaMemcpyAsync(ok.data(), d_ok, (size_t)n_xfers * 8, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    if (local != GRAPPA_OK) {
        set_error("%s", local_msg.c_str());
        return local;
    }
    for (int32_t k = 0; k < n_xfers; k++)
        GRAPPA_ARG(ok[k] == 1, GRAPPA_E_NCCL,
                   "grappa_shard_exchange: rank %d could not receive transfer %d (its own error says why)",
                   xfers[k].peer, k);
    // round 2: the arrays (sizes known on both sides from the header)
    SH_NCCL(ncclGroupStart());
    for (int32_t k = 0; k < n_xfers; k++) {
        const grappa_shard_info& I = xfers[k].send ? xfers[k].send->info : rs[k]->info;
        const int64_t esz = I.dtype == GRAPPA_BF16 ? 2 : 4;
        struct { const void* p; size_t bytes; } arr[6] = {
            {I.ids, (size_t)I.n_rows * 4}, {I.rowptr, (size_t)(I.n_rows + 1) * 8}, {I.col, (size_t)I.nnz * 4},
            {I.x, (size_t)I.n_rows * I.feat_dim * esz}, {I.labels, (size_t)I.n_rows * 4}, {I.train, (size_t)I.n_rows}};
        for (auto& a : arr) {
            if (a.bytes == 0) continue;
            if (xfers[k].send) {
                SH_NCCL(ncclSend(a.p, a.bytes, ncclUint8, xfers[k].peer, comm, s));
                if (xfers[k].peer != ctx->rank) ctx->comm_other_bytes += (int64_t)a.bytes;
            }
            else {
                SH_NCCL(ncclRecv(const_cast<void*>(a.p), a.bytes, ncclUint8, xfers[k].peer, comm, s));
            }
        }
    }
    SH_NCCL(ncclGroupEnd());
    return GRAPPA_OK;
}
