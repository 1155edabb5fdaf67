// halo.cu -- halo feature exchange of sharded halo-1 partitions (§8f row 2, second half).
//
// PAPER: P:410 (§4 "Halo node features are pre-cached at super-epoch boundaries"), P:413 ("load
// the new chunk's edges and synchronize halo features"), P:416 ("Feature gathering during
// repartitioning uses all-to-all collectives"); partitions with halo nodes P:177, P:196 (reading
// R33: core rows keep every neighbour, halo rows are empty and read-only).
//
// In sharded mode a rank holds only the chunk shards it owns.  A halo-1 partition built from its
// pair's two shards (grappa_repartition_shards_ex(GRAPPA_PART_HALO1)) knows its halo nodes --
// non-core neighbours of core rows, ascending global id (R34) -- but not their data: the halo
// node's features, global degree and label live in the shard of its chunk, on that chunk's owner.
// grappa_halo_exchange is the all-to-all that moves exactly those rows, once per partition build:
//   0. bucket the halo list by owner rank (stable: each bucket stays in ascending global id)
//   1. counts to every owner; one host sync sizes every buffer; 1b. an ok word back from every
//      server (both sides agree the buffers exist before any array moves: no unmatched sends)
//   2. the request ids to their owners
//   3. every server answers from its shards (binary search of the id in the shard's ascending
//      ids): feature row, global degree, label -- in request order
//   4. the replies back; the requester writes them into its halo rows (features, d_g, label, node
//      weight [d_g == 0]), which completes the partition: bitwise the replicated halo-1 partition.
// All of it is integer index work and byte copies.  Collective: every rank of the communicator
// calls it once per partition build in the same order, with or without a partition of its own.
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "part.cuh"
#include "scan.cuh"

namespace grappa {

struct HxFlagOwner {
    const int32_t* halo; const int32_t* chunk_of; const int32_t* owner; int32_t q;
    __device__ int32_t operator()(int64_t i) const { return owner[chunk_of[halo[i]]] == q; }
};
struct HxWriteReq {
    const int32_t* halo; int32_t* req_ids; int32_t* req_pos; int64_t base;
    __device__ void operator()(int64_t i, int64_t p, int32_t f) const {
        if (f) {
            req_ids[base + p] = halo[i];
            req_pos[base + p] = (int32_t)i;
        }
    }
    __device__ void finish(int64_t, int64_t) const {}
};

__global__ void k_hx_count(int64_t n, const int32_t* __restrict__ halo, const int32_t* __restrict__ chunk_of,
                           const int32_t* __restrict__ owner, int G, unsigned long long* __restrict__ cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[owner[chunk_of[halo[i]]]], 1ull);
}

struct HxShards {            // this rank's shards, by chunk (slot[c] = index or -1)
    const int32_t* ids[64];
    const int64_t* rowptr[64];
    const int32_t* labels[64];
    const uint4* x[64];
    int64_t n[64];
};

// answer requests: row of id u in its shard (ascending ids: binary search), its features (vec
// 16-byte vectors per row), global degree and label; bad[0] set if an id is not held here
__global__ void k_hx_serve(int64_t n_req, const int32_t* __restrict__ req, const int32_t* __restrict__ chunk_of,
                           const int32_t* __restrict__ slot, HxShards S, int64_t vec, uint4* __restrict__ rep_x,
                           int32_t* __restrict__ rep_deg, int32_t* __restrict__ rep_lab, int* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_req; k += nwarps) {
        const int32_t u = req[k];
        const int32_t sl = slot[chunk_of[u]];
        int64_t j = -1;
        if (sl >= 0) {
            int64_t lo = 0, hi = S.n[sl];
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (S.ids[sl][mid] < u) lo = mid + 1;
                else hi = mid;
            }
            if (lo < S.n[sl] && S.ids[sl][lo] == u) j = lo;
        }
        if (j < 0) {
            if (lane == 0) *bad = 1;
            continue;
        }
        for (int64_t t = lane; t < vec; t += 32) rep_x[k * vec + t] = S.x[sl][j * vec + t];
        if (lane == 0) {
            rep_deg[k] = (int32_t)(S.rowptr[sl][j + 1] - S.rowptr[sl][j]);
            rep_lab[k] = S.labels[sl][j];
        }
    }
}

// write the replies into the partition's halo rows (local row n_core + pos)
__global__ void k_hx_place(int64_t n, int64_t n_core, int64_t n_local, const int32_t* __restrict__ pos,
                           const uint4* __restrict__ rx, const int32_t* __restrict__ rdeg,
                           const int32_t* __restrict__ rlab, int64_t vec, uint4* __restrict__ x,
                           int32_t* __restrict__ d_g, int32_t* __restrict__ labels, float* __restrict__ node_w) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps) {
        const int64_t i = n_core + pos[k];
        for (int64_t t = lane; t < vec; t += 32) x[i * vec + t] = rx[k * vec + t];
        if (lane == 0) {
            const int32_t dg = rdeg[k];
            d_g[i] = dg;
            labels[i] = rlab[k];
            const float w = dg == 0 ? 1.0f : 0.0f;       // halo rows: d_l = 0 (k_halo_rows)
            node_w[i] = w;
            node_w[n_local + i] = w;
            node_w[2 * n_local + i] = 0.0f;
        }
    }
}

}  // namespace grappa

using namespace grappa;

#define HX_NCCL(expr)                                                                     \
    do {                                                                                  \
        ncclResult_t _r = (expr);                                                         \
        if (_r != ncclSuccess) {                                                          \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(_r)); \
            return GRAPPA_E_NCCL;                                                         \
        }                                                                                 \
    } while (0)

extern "C" grappa_status grappa_halo_exchange(grappa_ctx* ctx, grappa_part* part, int32_t n_shards,
                                              const grappa_shard* const* shards, const int32_t* chunk_owner,
                                              const int32_t* chunk_of, int32_t num_chunks, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && chunk_owner && chunk_of && (n_shards == 0 || shards), GRAPPA_E_ARG,
               "grappa_halo_exchange: null argument");
    // one rank without a communicator: every request is served locally (device copies)
    GRAPPA_ARG(ctx->comm || ctx->nranks == 1, GRAPPA_E_ARG, "grappa_halo_exchange: the ctx has no NCCL communicator");
    const bool local_only = !ctx->comm;
    GRAPPA_ARG(num_chunks >= 1 && num_chunks <= 64 && n_shards >= 0 && n_shards <= num_chunks, GRAPPA_E_ARG,
               "grappa_halo_exchange: 1 <= C <= 64 chunks, at most C shards");
    const int G = ctx->nranks;
    for (int c = 0; c < num_chunks; c++)
        GRAPPA_ARG(chunk_owner[c] >= 0 && chunk_owner[c] < G, GRAPPA_E_ARG,
                   "grappa_halo_exchange: chunk %d owner %d out of range", c, chunk_owner[c]);
    cudaStream_t s = (cudaStream_t)stream;
    ncclComm_t comm = (ncclComm_t)ctx->comm;
    // row format: from the partition, else from the shards this rank serves
    int32_t fd = -1;
    grappa_dtype dt = GRAPPA_F32;
    if (part) {
        GRAPPA_ARG(part->halo_pending || part->n_halo == 0 || !part->halo, GRAPPA_E_ARG,
                   "grappa_halo_exchange: partition is not a pending sharded halo-1 partition");
        fd = part->info.feat_dim;
        dt = part->info.dtype;
    }
    HxShards S{};
    std::vector<int32_t> slot(num_chunks, -1);
    for (int k = 0; k < n_shards; k++) {
        const grappa_shard_info& I = shards[k]->info;
        GRAPPA_ARG(I.chunk >= 0 && I.chunk < num_chunks && chunk_owner[I.chunk] == ctx->rank, GRAPPA_E_ARG,
                   "grappa_halo_exchange: shard of chunk %d is not owned by this rank", I.chunk);
        if (fd < 0) { fd = I.feat_dim; dt = I.dtype; }
        GRAPPA_ARG(I.feat_dim == fd && I.dtype == dt, GRAPPA_E_ARG,
                   "grappa_halo_exchange: shards / partition differ in feature width or dtype");
        slot[I.chunk] = k;
        S.ids[k] = I.ids; S.rowptr[k] = I.rowptr; S.labels[k] = I.labels; S.x[k] = (const uint4*)I.x; S.n[k] = I.n_rows;
    }
    if (fd < 0) fd = 0;
    const int64_t esz = dt == GRAPPA_BF16 ? 2 : 4;
    const int64_t row_bytes = (int64_t)fd * esz, vec = row_bytes / 16;
    const bool asks = part && part->halo_pending;
    const int64_t n_core = asks ? part->info.n_core - part->n_halo : 0;
    const int64_t n_halo = asks ? part->n_halo : 0;
    const int32_t* halo = asks ? (const int32_t*)part->core_global.p + n_core : nullptr;
    // small device tables: owner[C], slot[C], counts
    const size_t small_b = (size_t)num_chunks * 8 + (size_t)G * 16 + 64;
    GRAPPA_TRY(ctx->xf_hdr.grow(small_b + (size_t)G * 16));      // + the ok words of round 1b
    int32_t* d_owner = (int32_t*)ctx->xf_hdr.p;
    int32_t* d_slot = d_owner + num_chunks;
    int64_t* d_cnt = (int64_t*)((char*)ctx->xf_hdr.p + (size_t)num_chunks * 8);   // [G] mine to q
    int64_t* d_in = d_cnt + G;                                                     // [G] from r
    int* d_bad = (int*)(d_in + G);
    GRAPPA_CUDA(cudaMemcpyAsync(d_owner, chunk_owner, (size_t)num_chunks * 4, cudaMemcpyHostToDevice, s));
    GRAPPA_CUDA(cudaMemcpyAsync(d_slot, slot.data(), (size_t)num_chunks * 4, cudaMemcpyHostToDevice, s));
    GRAPPA_CUDA(cudaMemsetAsync(d_cnt, 0, (size_t)G * 8, s));
    GRAPPA_CUDA(cudaMemsetAsync(d_bad, 0, 4, s));
    // 0. per-owner request counts (exact integers)
    if (n_halo > 0) {
        k_hx_count<<<(unsigned)std::min<int64_t>(ceil_div(n_halo, 256), (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
            n_halo, halo, chunk_of, d_owner, G, (unsigned long long*)d_cnt);
        GRAPPA_LAUNCHED(ctx);
    }
    // 1. counts to every rank
    if (local_only) {
        GRAPPA_CUDA(cudaMemcpyAsync(d_in, d_cnt, 8, cudaMemcpyDeviceToDevice, s));
    } else {
        HX_NCCL(ncclGroupStart());
        for (int r = 0; r < G; r++) {
            HX_NCCL(ncclSend(d_cnt + r, 1, ncclInt64, r, comm, s));
            HX_NCCL(ncclRecv(d_in + r, 1, ncclInt64, r, comm, s));
        }
        HX_NCCL(ncclGroupEnd());
    }
    std::vector<int64_t> cnt(G), in(G);
    GRAPPA_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, (size_t)G * 8, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaMemcpyAsync(in.data(), d_in, (size_t)G * 8, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> qoff(G + 1, 0), roff(G + 1, 0);
    for (int q = 0; q < G; q++) qoff[q + 1] = qoff[q] + cnt[q];
    for (int r = 0; r < G; r++) roff[r + 1] = roff[r] + in[r];
    const int64_t n_req = qoff[G], n_srv = roff[G];
    // buffers: requests (ids, halo positions), served (ids in, replies out), received replies
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t b_rid = al((size_t)(n_req + 1) * 4), b_rpos = b_rid, b_sid = al((size_t)(n_srv + 1) * 4),
                 b_sx = al((size_t)(n_srv + 1) * row_bytes), b_sdeg = b_sid, b_slab = b_sid,
                 b_rx = al((size_t)(n_req + 1) * row_bytes), b_rdeg = b_rid, b_rlab = b_rid;
    grappa_status local = ctx->sh_ws.grow(b_rid + b_rpos + b_sid + b_sx + b_sdeg + b_slab + b_rx + b_rdeg + b_rlab);
    std::string local_msg = local == GRAPPA_OK ? "" : grappa_last_error();
    // 1b. every server tells every requester whether it can answer (so no send is left unmatched)
    int64_t* d_ok = (int64_t*)((char*)ctx->xf_hdr.p + small_b);
    std::vector<int64_t> ok_out(G, local == GRAPPA_OK ? 1 : 0), ok_in(G, 0);
    if (local_only) {
        ok_in = ok_out;
    } else {
        GRAPPA_CUDA(cudaMemcpyAsync(d_ok, ok_out.data(), (size_t)G * 8, cudaMemcpyHostToDevice, s));
        HX_NCCL(ncclGroupStart());
        for (int r = 0; r < G; r++) {
            HX_NCCL(ncclSend(d_ok, 1, ncclInt64, r, comm, s));
            HX_NCCL(ncclRecv(d_ok + G + r, 1, ncclInt64, r, comm, s));
        }
        HX_NCCL(ncclGroupEnd());
        GRAPPA_CUDA(cudaMemcpyAsync(ok_in.data(), d_ok + G, (size_t)G * 8, cudaMemcpyDeviceToHost, s));
        GRAPPA_CUDA(cudaStreamSynchronize(s));
    }
    if (local != GRAPPA_OK) {
        set_error("%s", local_msg.c_str());
        return local;
    }
    for (int r = 0; r < G; r++)
        GRAPPA_ARG(ok_in[r] == 1, GRAPPA_E_NCCL, "grappa_halo_exchange: rank %d could not take part (its own error "
                                                 "says why)", r);
    char* w = (char*)ctx->sh_ws.p;
    int32_t* rid = (int32_t*)w; w += b_rid;
    int32_t* rpos = (int32_t*)w; w += b_rpos;
    int32_t* sid = (int32_t*)w; w += b_sid;
    uint4* sx = (uint4*)w; w += b_sx;
    int32_t* sdeg = (int32_t*)w; w += b_sdeg;
    int32_t* slab = (int32_t*)w; w += b_slab;
    uint4* rx = (uint4*)w; w += b_rx;
    int32_t* rdeg = (int32_t*)w; w += b_rdeg;
    int32_t* rlab = (int32_t*)w;
    // 0b. stable buckets by owner (ascending global id inside each)
    for (int q = 0; q < G && n_halo > 0; q++)
        if (cnt[q]) GRAPPA_TRY(device_scan(ctx, HxFlagOwner{halo, chunk_of, d_owner, q}, n_halo,
                                           HxWriteReq{halo, rid, rpos, qoff[q]}, s));
    // 2. request ids to their owners
    if (local_only) {
        if (n_req) GRAPPA_CUDA(cudaMemcpyAsync(sid, rid, (size_t)n_req * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        HX_NCCL(ncclGroupStart());
        for (int r = 0; r < G; r++) {
            if (cnt[r]) HX_NCCL(ncclSend(rid + qoff[r], (size_t)cnt[r], ncclInt32, r, comm, s));
            if (in[r]) HX_NCCL(ncclRecv(sid + roff[r], (size_t)in[r], ncclInt32, r, comm, s));
            if (r != ctx->rank) ctx->comm_other_bytes += cnt[r] * 4;
        }
        HX_NCCL(ncclGroupEnd());
    }
    // 3. answer from this rank's shards
    if (n_srv > 0) {
        k_hx_serve<<<(unsigned)std::min<int64_t>(ceil_div(n_srv, 8), (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
            n_srv, sid, chunk_of, d_slot, S, vec, sx, sdeg, slab, d_bad);
        GRAPPA_LAUNCHED(ctx);
    }
    // 4. replies back
    if (local_only && n_req) {
        if (row_bytes) GRAPPA_CUDA(cudaMemcpyAsync(rx, sx, (size_t)(n_req * row_bytes), cudaMemcpyDeviceToDevice, s));
        GRAPPA_CUDA(cudaMemcpyAsync(rdeg, sdeg, (size_t)n_req * 4, cudaMemcpyDeviceToDevice, s));
        GRAPPA_CUDA(cudaMemcpyAsync(rlab, slab, (size_t)n_req * 4, cudaMemcpyDeviceToDevice, s));
    }
    if (!local_only) HX_NCCL(ncclGroupStart());
    for (int r = 0; r < G && !local_only; r++) {
        if (in[r]) {
            if (row_bytes) HX_NCCL(ncclSend(sx + roff[r] * vec, (size_t)(in[r] * row_bytes), ncclUint8, r, comm, s));
            HX_NCCL(ncclSend(sdeg + roff[r], (size_t)in[r], ncclInt32, r, comm, s));
            HX_NCCL(ncclSend(slab + roff[r], (size_t)in[r], ncclInt32, r, comm, s));
            if (r != ctx->rank) ctx->comm_other_bytes += in[r] * (row_bytes + 8);
        }
        if (cnt[r]) {
            if (row_bytes) HX_NCCL(ncclRecv(rx + qoff[r] * vec, (size_t)(cnt[r] * row_bytes), ncclUint8, r, comm, s));
            HX_NCCL(ncclRecv(rdeg + qoff[r], (size_t)cnt[r], ncclInt32, r, comm, s));
            HX_NCCL(ncclRecv(rlab + qoff[r], (size_t)cnt[r], ncclInt32, r, comm, s));
        }
    }
    if (!local_only) HX_NCCL(ncclGroupEnd());
    if (n_req > 0) {
        const int64_t n_local = part->info.n_core;
        k_hx_place<<<(unsigned)std::min<int64_t>(ceil_div(n_req, 8), (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
            n_req, n_core, n_local, rpos, rx, rdeg, rlab, vec, (uint4*)part->x.p, (int32_t*)part->d_g.p,
            (int32_t*)part->labels.p, (float*)part->node_w.p);
        GRAPPA_LAUNCHED(ctx);
    }
    // every rank learns whether any server met a request it does not hold (the requester's halo
    // rows would otherwise hold whatever that server sent)
    if (!local_only) HX_NCCL(ncclAllReduce(d_bad, d_bad, 1, ncclInt32, ncclMax, comm, s));
    int bad = 0;
    GRAPPA_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    GRAPPA_ARG(!bad, GRAPPA_E_ARG,
               "grappa_halo_exchange: a requested halo node is not in its owner's shards (on some rank)");
    if (part) part->halo_pending = false;
    return GRAPPA_OK;
}
