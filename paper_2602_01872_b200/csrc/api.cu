// api.cu -- context, error plumbing, layer orchestration (a4/a6) and gradient aggregation
// (a7/a8) of the grappa C ABI.  See include/grappa.h for the contract of every entry point.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <nccl.h>

#include "gemm.cuh"
#include "part.cuh"
#include "spmm.cuh"

namespace grappa {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static thread_local std::shared_ptr<const Allocator> tl_alloc;
static thread_local void* tl_stream = nullptr;

CallScope::CallScope(const grappa_ctx* ctx, void* stream) : prev_al(tl_alloc), prev_stream(tl_stream) {
    tl_alloc = ctx ? ctx->alloc : nullptr;
    tl_stream = stream;
}
CallScope::~CallScope() {
    tl_alloc = prev_al;
    tl_stream = prev_stream;
}

grappa_status DevBuf::grow(size_t bytes) {
    if (bytes <= cap && p) return GRAPPA_OK;
    release();
    // 1/8 headroom: partition sizes fluctuate by a few % across super-epochs, and a realloc
    // inside a switch is what we want to avoid
    size_t b = bytes < 256 ? 256 : bytes + bytes / 8;
    std::shared_ptr<const Allocator> a = tl_alloc;
    if (a) {
        // a caller pool bound to a stream under graph capture would tie the block to the graph
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing((cudaStream_t)tl_stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
            a = nullptr;
    }
    if (a) {
        p = a->alloc(b, tl_stream, a->user);
        if (!p) {
            set_error("caller allocator failed for %zu bytes", b);
            return GRAPPA_E_NOMEM;
        }
        al = a;
        al_stream = tl_stream;
    } else {
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            p = nullptr;
            set_error("cudaMalloc(%zu): %s", b, cudaGetErrorString(e));
            return GRAPPA_E_NOMEM;
        }
        al = nullptr;
    }
    cap = b;
    return GRAPPA_OK;
}

void DevBuf::release() {
    if (p) {
        if (al) al->free(p, cap, al_stream, al->user);
        else cudaFree(p);
    }
    p = nullptr;
    cap = 0;
    al = nullptr;
}

static cudaEvent_t take_event(grappa_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(grappa_ctx* c, cudaStream_t st, int cls, double bytes, double flops)
    : ctx(c), s(st) {
    if (!ctx || !ctx->profiling) return;
    ProfRec r{take_event(ctx), take_event(ctx), cls, bytes, flops};
    cudaEventRecord(r.a, s);
    idx = (int)ctx->prof.size();
    ctx->prof.push_back(r);
}

void ProfScope::set_bytes(double bytes) {
    if (idx >= 0) ctx->prof[idx].bytes = bytes;
}

ProfScope::~ProfScope() {
    if (idx >= 0) cudaEventRecord(ctx->prof[idx].b, s);
}

}  // namespace grappa

using namespace grappa;

#define NCCL_OK(expr)                                                                 \
    do {                                                                              \
        ncclResult_t _r = (expr);                                                     \
        if (_r != ncclSuccess) {                                                      \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(_r)); \
            return GRAPPA_E_NCCL;                                                     \
        }                                                                             \
    } while (0)

extern "C" const char* grappa_version(void) { return "grappa-b200 0.1 (sm_100a)"; }
extern "C" const char* grappa_last_error(void) { return g_err; }

extern "C" grappa_status grappa_nccl_unique_id(void* out128) {
    GRAPPA_ARG(out128, GRAPPA_E_ARG, "grappa_nccl_unique_id: null");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NCCL_OK(ncclGetUniqueId(&id));
    memcpy(out128, &id, 128);
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_ctx_create(int device, const void* nccl_uid, int rank, int nranks,
                                           grappa_ctx** out) {
    return grappa_ctx_create_ex(device, nccl_uid, rank, nranks, nullptr, nullptr, nullptr, out);
}

extern "C" grappa_status grappa_ctx_create_ex(int device, const void* nccl_uid, int rank, int nranks,
                                              grappa_alloc_fn alloc, grappa_free_fn free_fn, void* alloc_user,
                                              grappa_ctx** out) {
    GRAPPA_ARG(out, GRAPPA_E_ARG, "grappa_ctx_create: null out");
    GRAPPA_ARG(nranks >= 1 && rank >= 0 && rank < nranks, GRAPPA_E_ARG,
               "grappa_ctx_create: bad rank %d / nranks %d", rank, nranks);
    GRAPPA_CUDA(cudaSetDevice(device));
    grappa_ctx* c = new grappa_ctx();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    if (alloc && free_fn) {
        auto a = std::make_shared<Allocator>();
        a->alloc = alloc;
        a->free = free_fn;
        a->user = alloc_user;
        c->alloc = a;
    }
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess || cudaMemset(c->d_flag, 0, sizeof(int)) != cudaSuccess) {
        delete c;
        set_error("grappa_ctx_create: cannot allocate flag");
        return GRAPPA_E_NOMEM;
    }
    if (nccl_uid) {   // a 1-rank communicator serves the shard exchange's self transfers
        ncclUniqueId id;
        memcpy(&id, nccl_uid, 128);
        ncclComm_t comm;
        ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
        if (r != ncclSuccess) {
            set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
            cudaFree(c->d_flag);
            delete c;
            return GRAPPA_E_NCCL;
        }
        c->comm = comm;
    }
    *out = c;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_comm_bytes(const grappa_ctx* ctx, int64_t* grad_bytes, int64_t* other_bytes) {
    GRAPPA_ARG(ctx && grad_bytes && other_bytes, GRAPPA_E_ARG, "grappa_comm_bytes: null argument");
    *grad_bytes = ctx->comm_grad_bytes;
    *other_bytes = ctx->comm_other_bytes;
    return GRAPPA_OK;
}

extern "C" void grappa_ctx_destroy(grappa_ctx* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy((ncclComm_t)c->comm);
    c->scan_ws.release();
    c->red_ws.release();
    c->small.release();
    c->rp_ws.release();
    c->sh_ws.release();
    c->xf_hdr.release();
    c->comm_buf.release();
    c->wimg.release();
    c->loss_ws.release();
    for (int i = 0; i < grappa_ctx::kRpStreams; i++) {
        c->rp_scan[i].release();
        c->rp_small[i].release();
        c->rp_rank[i].release();
        if (c->rp_s[i]) cudaStreamDestroy(c->rp_s[i]);
    }
    for (int i = 0; i <= grappa_ctx::kRpStreams; i++)
        if (c->rp_ev[i]) cudaEventDestroy(c->rp_ev[i]);
    for (auto& r : c->prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->d_flag) cudaFree(c->d_flag);
    delete c;
}

extern "C" int64_t grappa_launch_count(const grappa_ctx* c) { return c ? c->launches : 0; }

extern "C" grappa_status grappa_set_kernel_variant(grappa_ctx* ctx, const char* op, int variant) {
    GRAPPA_ARG(ctx && op, GRAPPA_E_ARG, "grappa_set_kernel_variant: null argument");
    if (!strcmp(op, "gemm") && variant >= 0 && variant <= 2) { ctx->var_gemm = variant; return GRAPPA_OK; }
    if (!strcmp(op, "spmm") && variant >= 0 && variant <= 5) { ctx->var_spmm = variant; return GRAPPA_OK; }
    if (!strcmp(op, "pair") && variant >= 0 && variant <= 1) { ctx->var_pair = variant; return GRAPPA_OK; }
    if (!strcmp(op, "wstream") && variant >= 0 && variant <= 2) { ctx->var_gemm_stream = variant; return GRAPPA_OK; }
    set_error("grappa_set_kernel_variant: unknown op '%s' or variant %d", op, variant);
    return GRAPPA_E_ARG;
}

extern "C" grappa_status grappa_profile_enable(grappa_ctx* c, int on) {
    GRAPPA_ARG(c, GRAPPA_E_ARG, "grappa_profile_enable: null ctx");
    for (auto& r : c->prof) {
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->prof.clear();
    c->profiling = on != 0;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_profile_read(grappa_ctx* c, int cls, double* ms, int64_t* calls,
                                             double* bytes, double* flops) {
    GRAPPA_ARG(c && ms && calls && bytes && flops, GRAPPA_E_ARG, "grappa_profile_read: null argument");
    double t = 0, by = 0, fl = 0;
    int64_t n = 0;
    for (auto& r : c->prof) {
        if (r.cls != cls) continue;
        GRAPPA_CUDA(cudaEventSynchronize(r.b));
        float e = 0.f;
        GRAPPA_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
        t += e; by += r.bytes; fl += r.flops; n++;
    }
    *ms = t; *calls = n; *bytes = by; *flops = fl;
    return GRAPPA_OK;
}

// ------------------------------------------------------------------------------ layers
static inline size_t esz_of(grappa_dtype dt) { return dt == GRAPPA_BF16 ? 2 : 4; }

namespace grappa {
size_t gat_saved_bytes(const grappa_part* part, int f_out, grappa_dtype dt);
size_t gat_ws_bytes(const grappa_part* part, int f_in, int f_out, grappa_dtype dt);
grappa_status gat_fwd(grappa_ctx* ctx, const grappa_part* part, int f_in, int f_out, int relu, const void* h_in,
                      const float* w, void* h_out, void* saved, void* ws, grappa_dtype dt, cudaStream_t s);
grappa_status gat_bwd(grappa_ctx* ctx, const grappa_part* part, int f_in, int f_out, int relu_in,
                      const void* dz_out, const void* h_in, const float* w, const void* saved, float* dw,
                      void* dz_in, void* ws, grappa_dtype dt, cudaStream_t s);
}  // namespace grappa

extern "C" size_t grappa_layer_saved_bytes_ex(const grappa_part* part, grappa_arch arch, int32_t f_in,
                                              int32_t f_out, grappa_dtype dtype, unsigned flags) {
    if (part && arch == GRAPPA_GCN && (flags & GRAPPA_LAYER_INPUT))
        return (size_t)part->info.n_core * f_in * esz_of(dtype);   // P = Ahat h_in (aggregate-first)
    return grappa_layer_saved_bytes(part, arch, f_in, f_out, dtype);
}

extern "C" size_t grappa_layer_saved_bytes(const grappa_part* part, grappa_arch arch, int32_t f_in,
                                           int32_t f_out, grappa_dtype dtype) {
    if (part && arch == GRAPPA_GAT) return gat_saved_bytes(part, f_out, dtype);
    if (!part || arch != GRAPPA_SAGE) return 0;
    return (size_t)part->info.n_core * f_in * esz_of(dtype);   // M = D^-1 A h_in
}

extern "C" size_t grappa_layer_ws_bytes(const grappa_part* part, grappa_arch arch, int32_t f_in,
                                        int32_t f_out, grappa_dtype dtype) {
    if (!part) return 0;
    if (arch == GRAPPA_GAT) return gat_ws_bytes(part, f_in, f_out, dtype);
    const int64_t n = part->info.n_core, slots = std::max<int64_t>(part->info.n_slots, part->t_n_slots);
    const size_t es = esz_of(dtype);
    const int wmax = f_in > f_out ? f_in : f_out;
    // T / dT / dM; GCN: also the input layer's pre-scaled rows N h_in (width f_in)
    size_t node = (size_t)n * (arch == GRAPPA_GCN ? wmax : f_in) * es;
    size_t partial = (size_t)slots * wmax * 4;
    size_t splitk = gemm_tn_ws_bytes(n, f_in, arch == GRAPPA_GCN ? 0 : f_in, f_out);
    // GCN node-level backward: the pre-weighted rows w_u dz_u (R30c)
    size_t node2 = arch == GRAPPA_GCN ? (size_t)n * f_out * es : 0;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    return al(node) + al(partial) + al(splitk) + al(node2);
}

struct WsLayout {
    void* node;
    float* partial;
    float* splitk;
    void* node2;
};
static WsLayout carve(const grappa_part* part, grappa_arch arch, int f_in, int f_out,
                      grappa_dtype dt, void* ws) {
    const int64_t n = part->info.n_core, slots = std::max<int64_t>(part->info.n_slots, part->t_n_slots);
    const size_t es = esz_of(dt);
    const int wmax = f_in > f_out ? f_in : f_out;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    size_t node = al((size_t)n * (arch == GRAPPA_GCN ? wmax : f_in) * es);   // as grappa_layer_ws_bytes
    size_t partial = al((size_t)slots * wmax * 4);
    size_t splitk = al(gemm_tn_ws_bytes(n, f_in, arch == GRAPPA_GCN ? 0 : f_in, f_out));
    char* b = (char*)ws;
    return WsLayout{b, (float*)(b + node), (float*)(b + node + partial), b + node + partial + splitk};
}

static grappa_status check_dims(const char* who, int f_in, int f_out) {
    GRAPPA_ARG(f_in > 0 && f_out > 0 && f_in % 16 == 0 && f_out % 16 == 0, GRAPPA_E_SHAPE,
               "%s: f_in=%d f_out=%d must be positive multiples of 16", who, f_in, f_out);
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_layer_fwd(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                          int32_t f_in, int32_t f_out, int relu, const void* h_in,
                                          const float* w, void* h_out, void* saved, void* ws,
                                          grappa_dtype dtype, void* stream) {
    CallScope call_scope(ctx, stream);
    return grappa_layer_fwd_ex(ctx, part, arch, f_in, f_out, relu, h_in, w, h_out, saved, ws, dtype, 0u,
                               stream);
}

extern "C" grappa_status grappa_layer_fwd_ex(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                             int32_t f_in, int32_t f_out, int relu, const void* h_in,
                                             const float* w, void* h_out, void* saved, void* ws,
                                             grappa_dtype dtype, unsigned flags, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG((flags & ~(GRAPPA_LAYER_NODE_LEVEL | GRAPPA_LAYER_INPUT)) == 0, GRAPPA_E_ARG,
               "grappa_layer_fwd_ex: flags 0x%x invalid", flags);
    GRAPPA_ARG(arch != GRAPPA_GCN || !(flags & GRAPPA_LAYER_INPUT) || saved, GRAPPA_E_ARG,
               "grappa_layer_fwd_ex: GRAPPA_LAYER_INPUT (GCN) needs `saved` (grappa_layer_saved_bytes_ex)");
    GRAPPA_ARG(ctx && part && h_in && w && h_out && ws, GRAPPA_E_ARG, "grappa_layer_fwd: null argument");
    GRAPPA_ARG(!part->halo_pending, GRAPPA_E_ARG,
               "grappa_layer_fwd: the partition's halo rows are pending (grappa_halo_exchange first)");
    GRAPPA_TRY(check_dims("grappa_layer_fwd", f_in, f_out));
    GRAPPA_ARG(arch == GRAPPA_GCN || saved, GRAPPA_E_ARG, "grappa_layer_fwd: SAGE / GAT need `saved`");
    GRAPPA_ARG(arch == GRAPPA_GCN || arch == GRAPPA_SAGE || arch == GRAPPA_GAT, GRAPPA_E_ARG,
               "grappa_layer_fwd: unknown arch %d", (int)arch);
    cudaStream_t s = (cudaStream_t)stream;
    const grappa_part_info& I = part->info;
    const bool node = flags & GRAPPA_LAYER_NODE_LEVEL;
    if (arch == GRAPPA_GAT) {
        GRAPPA_ARG(!node, GRAPPA_E_ARG, "grappa_layer_fwd_ex: node-level weights are not defined for GAT (R35)");
        return gat_fwd(ctx, part, f_in, f_out, relu, h_in, w, h_out, saved, ws, dtype, s);
    }
    const float* w_node = node ? I.node_w : nullptr;                       // w_v
    const float* sage_scale = node ? I.node_w + 2 * I.n_core : I.norm_sage;  // w_v / d_l
    WsLayout L = carve(part, arch, f_in, f_out, dtype, ws);
    if (arch == GRAPPA_GCN && (flags & GRAPPA_LAYER_INPUT)) {
        // input layer, aggregate-first: P = Ahat h_in (kept in `saved`), h_out = act(P W); its
        // backward is then dW = P^T dz with no aggregation at all (no dh_in for the input)
        // (R29c) the source normalisation is applied once per row, h' = N h_in rounded to the
        // storage dtype, so the aggregation gathers unweighted rows: P = N (h'_v + sum h'_u)
        GRAPPA_TRY(row_scale(ctx, h_in, I.n_core, f_in, I.norm_gcn, L.node, dtype, s));
        SpmmArgs a;
        a.X = L.node; a.width = f_in; a.row_scale = I.norm_gcn; a.col_scale = nullptr; a.nbr_scale = w_node;
        a.self = 1; a.out = saved; a.partial = L.partial;
        GRAPPA_TRY(spmm(ctx, part, a, dtype, s));
        GemmArgs g;
        g.M = I.n_core; g.K1 = f_in; g.N = f_out; g.A1 = saved; g.B = w; g.relu = relu; g.n_split = f_out;
        g.C1 = h_out;
        return gemm_nn(ctx, g, dtype, s);
    }
    if (arch == GRAPPA_GCN) {
        // T = h_in W  (transform first: SpMM width = f_out)
        GemmArgs g;
        g.M = I.n_core; g.K1 = f_in; g.N = f_out; g.A1 = h_in; g.B = w;
        g.n_split = f_out; g.C1 = L.node;
        // the column normalisation n_u is applied once per row in the GEMM epilogue
        // (T' = N T), so the SpMM gathers unweighted rows (no per-edge scale load)
        g.row_scale = I.norm_gcn;
        GRAPPA_TRY(gemm_nn(ctx, g, dtype, s));
        // h_out = act(n_v (T'_v + sum T'_u)) = act(n_v (n_v T_v + sum n_u T_u))
        // node-level: act(n_v (T'_v + w_v sum T'_u))
        SpmmArgs a;
        a.X = L.node; a.width = f_out; a.row_scale = I.norm_gcn; a.col_scale = nullptr;
        a.nbr_scale = w_node;
        a.self = 1; a.relu = relu; a.out = h_out; a.partial = L.partial;
        return spmm(ctx, part, a, dtype, s);
    }
    // SAGE: M = D^-1 A h_in (node-level: diag(w) D^-1 A h_in) ; h_out = act([h_in | M] [Ws; Wn])
    SpmmArgs a;
    a.X = h_in; a.width = f_in; a.row_scale = sage_scale; a.out = saved; a.partial = L.partial;
    GRAPPA_TRY(spmm(ctx, part, a, dtype, s));
    GemmArgs g;
    g.M = I.n_core; g.K1 = f_in; g.K2 = f_in; g.N = f_out; g.A1 = h_in; g.A2 = saved; g.B = w;
    g.relu = relu; g.n_split = f_out; g.C1 = h_out;
    return gemm_nn(ctx, g, dtype, s);
}

extern "C" grappa_status grappa_layer_bwd(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                          int32_t f_in, int32_t f_out, int relu_in, const void* dz_out,
                                          const void* h_in, const float* w, const void* saved,
                                          float* dw, void* dz_in, void* ws, grappa_dtype dtype,
                                          void* stream) {
    CallScope call_scope(ctx, stream);
    return grappa_layer_bwd_ex(ctx, part, arch, f_in, f_out, relu_in, dz_out, h_in, w, saved, dw, dz_in,
                               ws, dtype, 0u, stream);
}

extern "C" grappa_status grappa_layer_bwd_ex(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                             int32_t f_in, int32_t f_out, int relu_in, const void* dz_out,
                                             const void* h_in, const float* w, const void* saved,
                                             float* dw, void* dz_in, void* ws, grappa_dtype dtype,
                                             unsigned flags, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG((flags & ~(3u | GRAPPA_LAYER_NODE_LEVEL | GRAPPA_LAYER_INPUT)) == 0 &&
                   ((flags & 3u) == 0 || arch == GRAPPA_GCN),
               GRAPPA_E_ARG, "grappa_layer_bwd_ex: flags 0x%x invalid (normalised gradients are GCN-only)", flags);
    const bool out_normed = flags & GRAPPA_BWD_DZ_OUT_NORMED, in_normed = flags & GRAPPA_BWD_DZ_IN_NORMED;
    const bool node = flags & GRAPPA_LAYER_NODE_LEVEL;
    GRAPPA_ARG(ctx && part && dz_out && h_in && w && dw && ws, GRAPPA_E_ARG,
               "grappa_layer_bwd: null argument");
    GRAPPA_TRY(check_dims("grappa_layer_bwd", f_in, f_out));
    GRAPPA_ARG(arch == GRAPPA_GCN || saved, GRAPPA_E_ARG, "grappa_layer_bwd: SAGE / GAT need `saved`");
    GRAPPA_ARG(arch == GRAPPA_GCN || arch == GRAPPA_SAGE || arch == GRAPPA_GAT, GRAPPA_E_ARG,
               "grappa_layer_bwd: unknown arch %d", (int)arch);
    cudaStream_t s = (cudaStream_t)stream;
    const grappa_part_info& I = part->info;
    if (arch == GRAPPA_GAT) {
        GRAPPA_ARG(!node, GRAPPA_E_ARG, "grappa_layer_bwd_ex: node-level weights are not defined for GAT (R35)");
        return gat_bwd(ctx, part, f_in, f_out, relu_in, dz_out, h_in, w, saved, dw, dz_in, ws, dtype, s);
    }
    if (arch == GRAPPA_GCN && (flags & GRAPPA_LAYER_INPUT)) {
        GRAPPA_ARG(!dz_in && !(flags & 3u) && saved, GRAPPA_E_ARG,
                   "grappa_layer_bwd_ex: GRAPPA_LAYER_INPUT takes no dz_in, no normalised flags, and the "
                   "forward's `saved`");
        GemmTNArgs t;
        t.M = I.n_core; t.K1 = f_in; t.N = f_out; t.A1 = saved; t.B = dz_out; t.C = dw;
        t.ws = carve(part, arch, f_in, f_out, dtype, ws).splitk;
        return gemm_tn(ctx, t, dtype, s);
    }
    WsLayout L = carve(part, arch, f_in, f_out, dtype, ws);
    if (arch == GRAPPA_GCN) {
        // dT = Ahat dz_out = N (A + I) (N dz_out): with a pre-normalised dz_out the SpMM
        // gathers unweighted rows.  Node-level (R30): Ahat_w^T dz = N (A diag(w) + I) (N dz) --
        // neighbours gathered with scale w_u (w_u n_u unnormalised), self term unweighted
        SpmmArgs a;
        a.X = dz_out; a.width = f_out; a.row_scale = I.norm_gcn; a.col_scale = out_normed ? nullptr : I.norm_gcn;
        if (node) {
            // (R30c) the neighbour weight w_u (w_u n_u unnormalised) is applied once per row:
            // dz' = w dz rounded to the storage dtype, gathered unweighted; the self term reads
            // the unweighted dz_v
            GRAPPA_TRY(row_scale(ctx, dz_out, I.n_core, f_out, out_normed ? I.node_w : I.node_w + I.n_core,
                                 L.node2, dtype, s));
            a.X = L.node2;
            a.X_self = dz_out;
            a.col_scale = nullptr;
            a.self_sep = 1;
            a.self_scale = out_normed ? nullptr : I.norm_gcn;
        }
        a.self = 1; a.out = L.node; a.partial = L.partial;
        GRAPPA_TRY(spmm_t(ctx, part, a, dtype, s));          // transpose operator (halo-1, R33)
        if (dz_in && dtype == GRAPPA_BF16 && !ctx->var_pair && gemm_tc_pair_supported(I.n_core, f_in, f_out)) {
            // both backward GEMMs from one read of dT and h_in (dz_in with the relu' gate, dW)
            const double M = (double)I.n_core;
            ProfScope ps(ctx, s, GRAPPA_K_GEMM, M * (f_out + 2.0 * f_in) * 2.0 + 4.0 * f_in * f_out * 2.0 +
                                                    (in_normed ? 4.0 * M : 0.0),
                         4.0 * M * f_in * f_out);
            return gemm_tc_pair(ctx, I.n_core, f_in, f_out, L.node, h_in, w, in_normed ? I.norm_gcn : nullptr,
                                relu_in, dz_in, L.splitk, dw, s);
        }
        // dW = h_in^T dT
        GemmTNArgs t;
        t.M = I.n_core; t.K1 = f_in; t.N = f_out; t.A1 = h_in; t.B = L.node; t.C = dw; t.ws = L.splitk;
        GRAPPA_TRY(gemm_tn(ctx, t, dtype, s));
        if (!dz_in) return GRAPPA_OK;
        // dz_in = (dT W^T) * relu'(h_in)
        GemmArgs g;
        g.M = I.n_core; g.K1 = f_out; g.N = f_in; g.A1 = L.node; g.B = w; g.b_trans = 1;
        g.mask = relu_in ? h_in : nullptr; g.n_split = f_in; g.C1 = dz_in;
        if (in_normed) g.row_scale = I.norm_gcn;          // write N dz_in
        return gemm_nn(ctx, g, dtype, s);
    }
    // SAGE: [dWs; dWn] = [h_in | M]^T dz_out
    GemmTNArgs t;
    t.M = I.n_core; t.K1 = f_in; t.K2 = f_in; t.N = f_out; t.A1 = h_in; t.A2 = saved; t.B = dz_out;
    t.C = dw; t.ws = L.splitk;
    GRAPPA_TRY(gemm_tn(ctx, t, dtype, s));
    if (!dz_in) return GRAPPA_OK;
    // [dh_s | dM] = dz_out [Ws^T | Wn^T];  dz_in = (dh_s + A D^-1 dM) * relu'(h_in)
    GemmArgs g;
    g.M = I.n_core; g.K1 = f_out; g.N = 2 * f_in; g.A1 = dz_out; g.B = w; g.b_trans = 1;
    g.n_split = f_in; g.C1 = dz_in; g.C2 = L.node;
    GRAPPA_TRY(gemm_nn(ctx, g, dtype, s));
    SpmmArgs a;
    a.X = L.node; a.width = f_in; a.col_scale = node ? I.node_w + 2 * I.n_core : I.norm_sage; a.accumulate = 1;
    a.mask = relu_in ? h_in : nullptr; a.out = dz_in; a.partial = L.partial;
    return spmm_t(ctx, part, a, dtype, s);
}

// ------------------------------------------------------------------------------ aggregate
namespace grappa {

// one fused pass before the all-reduce: comm = scale * grad (fp32 in place, or bf16 into
// the comm buffer); flags a non-finite scaled value
template <typename C>
__global__ void k_scale_grad(int64_t n, float* __restrict__ grad, float scale, C* __restrict__ comm, int* flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float g = grad[i] * scale;
        bad |= !isfinite(g);
        if constexpr (sizeof(C) == 4) grad[i] = g;
        else comm[i] = __float2bfloat16_rn(g);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// after the all-reduce: non-finite values that arrived from other ranks (or overflowed in the sum)
template <typename C>
__global__ void k_flag_nonfinite(int64_t n, const C* __restrict__ v, int* flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float g;
        if constexpr (sizeof(C) == 4) g = v[i];
        else g = __bfloat162float(v[i]);
        bad |= !isfinite(g);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// grad <- the aggregated value (bf16 comm buffer upcast; nothing for fp32) and, unless the flag is
// set (a non-finite aggregate in this or an earlier unchecked step), theta -= lr * grad
template <typename C>
__global__ void k_finish_sgd(int64_t n, const C* __restrict__ comm, float* __restrict__ grad, float lr,
                             float* __restrict__ theta, const int* __restrict__ flag) {
    const bool skip = *(volatile const int*)flag != 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float g;
        if constexpr (sizeof(C) == 4) {
            g = grad[i];
        } else {
            g = __bfloat162float(comm[i]);
            grad[i] = g;
        }
        if (theta && !skip) theta[i] = theta[i] - lr * g;
    }
}

static double factor_of(const grappa_part_info& I, grappa_corr corr, double eps, double c_max, bool* ok) {
    *ok = true;
    switch (corr) {
        case GRAPPA_CORR_NONE: return 1.0;
        case GRAPPA_CORR_NODE: return 1.0;          // correction inside the gradient (R30)
        case GRAPPA_CORR_UNIFORM: return I.c_uniform;
        case GRAPPA_CORR_RESAMPLING: {
            // full-graph: D = sum_{seeds, d_l>0} (d_g - d_l) exactly (s_v = d_l); R12 guards
            const double D = (double)I.D;
            return D < eps ? 1.0 : std::min(1.0 / D, c_max);
        }
        case GRAPPA_CORR_RESAMPLING_HM: return I.c_resampling_hm;
        default: *ok = false; return 0.0;
    }
}

}  // namespace grappa

extern "C" grappa_status grappa_aggregate_grads(grappa_ctx* ctx, const grappa_part* part, grappa_corr corr,
                                                double eps, double c_max, float* grad, int64_t n_params,
                                                int32_t m_active, grappa_dtype comm_dtype, float lr, float* theta,
                                                void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && grad && n_params > 0, GRAPPA_E_ARG, "grappa_aggregate_grads: null argument");
    GRAPPA_ARG(eps > 0.0 && c_max >= 1.0, GRAPPA_E_ARG,
               "grappa_aggregate_grads: need eps > 0 and c_max >= 1 (S:311-314), got %g / %g", eps, c_max);
    double c = 0.0;   // inactive rank: contributes zeros
    if (part) {
        bool ok;
        c = factor_of(part->info, corr, eps, c_max, &ok);
        GRAPPA_ARG(ok, GRAPPA_E_ARG, "grappa_aggregate_grads: bad corr %d", (int)corr);
        GRAPPA_ARG(std::isfinite(c), GRAPPA_E_NONFINITE, "grappa_aggregate_grads: non-finite c (S:361)");
    }
    return grappa_aggregate_grads_c(ctx, c, grad, n_params, m_active, comm_dtype, lr, theta, stream);
}

extern "C" grappa_status grappa_aggregate_grads_c(grappa_ctx* ctx, double c, float* grad, int64_t n_params,
                                                  int32_t m_active, grappa_dtype comm_dtype, float lr, float* theta,
                                                  void* stream) {
    CallScope scope(ctx, stream);
    GRAPPA_ARG(ctx && grad && n_params > 0, GRAPPA_E_ARG, "grappa_aggregate_grads_c: null argument");
    GRAPPA_ARG(m_active >= 1, GRAPPA_E_ARG, "grappa_aggregate_grads_c: m_active must be >= 1");
    GRAPPA_ARG(lr == 0.f || theta, GRAPPA_E_ARG, "grappa_aggregate_grads_c: lr != 0 needs theta");
    GRAPPA_ARG(comm_dtype == GRAPPA_F32 || comm_dtype == GRAPPA_BF16, GRAPPA_E_ARG,
               "grappa_aggregate_grads_c: bad comm_dtype %d", (int)comm_dtype);
    GRAPPA_ARG(std::isfinite(c), GRAPPA_E_NONFINITE, "grappa_aggregate_grads_c: non-finite c (S:361)");
    cudaStream_t s = (cudaStream_t)stream;
    const float scale = (float)(c / (double)m_active);
    const bool multi = ctx->comm && ctx->nranks > 1;
    const bool bf = comm_dtype == GRAPPA_BF16;
    const size_t cbytes = (size_t)n_params * (bf ? 2 : 4);
    if (bf) GRAPPA_TRY(ctx->comm_buf.grow(cbytes));
    __nv_bfloat16* cb = bf ? (__nv_bfloat16*)ctx->comm_buf.p : nullptr;
    ProfScope ps(ctx, s, GRAPPA_K_AGG, (double)n_params * (4.0 + (bf ? 2.0 : 4.0) + (lr != 0.f ? 12.0 : 0.0)),
                 3.0 * n_params);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n_params, 256), (int64_t)ctx->sm_count * 4);
    if (bf) k_scale_grad<__nv_bfloat16><<<grid, 256, 0, s>>>(n_params, grad, scale, cb, ctx->d_flag);
    else k_scale_grad<float><<<grid, 256, 0, s>>>(n_params, grad, scale, nullptr, ctx->d_flag);
    GRAPPA_LAUNCHED(ctx);
    if (multi) {
        NCCL_OK(ncclAllReduce(bf ? (void*)cb : (void*)grad, bf ? (void*)cb : (void*)grad, (size_t)n_params,
                              bf ? ncclBfloat16 : ncclFloat32, ncclSum, (ncclComm_t)ctx->comm, s));
        ctx->comm_grad_bytes += (int64_t)cbytes;
        if (bf) k_flag_nonfinite<__nv_bfloat16><<<grid, 256, 0, s>>>(n_params, cb, ctx->d_flag);
        else k_flag_nonfinite<float><<<grid, 256, 0, s>>>(n_params, grad, ctx->d_flag);
        GRAPPA_LAUNCHED(ctx);
    }
    if (bf || lr != 0.f) {
        if (bf) k_finish_sgd<__nv_bfloat16><<<grid, 256, 0, s>>>(n_params, cb, grad, lr, lr != 0.f ? theta : nullptr,
                                                                 ctx->d_flag);
        else k_finish_sgd<float><<<grid, 256, 0, s>>>(n_params, nullptr, grad, lr, theta, ctx->d_flag);
        GRAPPA_LAUNCHED(ctx);
    }
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_check(grappa_ctx* ctx, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx, GRAPPA_E_ARG, "grappa_check: null ctx");
    cudaStream_t s = (cudaStream_t)stream;
    int flag = 0;
    GRAPPA_CUDA(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GRAPPA_CUDA(cudaStreamSynchronize(s));
    if (ctx->comm) {
        ncclResult_t ar;
        NCCL_OK(ncclCommGetAsyncError((ncclComm_t)ctx->comm, &ar));
        NCCL_OK(ar);
    }
    if (flag) {
        GRAPPA_CUDA(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), s));
        set_error("non-finite aggregated gradient (S:424)");
        return GRAPPA_E_NONFINITE;
    }
    return GRAPPA_OK;
}
