// shard_host.cu -- host images of chunk shards: the data loader of capacity mode from chunk
// shards (§8f row 3; Alg. 1 with M < P beyond HBM).
//
// PAPER: P:196-198 (§3.3: nodes are assigned to chunks once; a partition = base chunk + swept
// chunk), P:395 ("trades training time for memory capacity"), P:410 (§4: partitions live in CPU
// memory and are loaded onto the GPU), P:656 (RMAT-36 trained one partition at a time).
//
// A chunk shard (the grappa_shard of sharded mode) holds one chunk's rows: its nodes in
// ascending global id, their full adjacency lists (global neighbour ids), features in the
// storage dtype, labels and train flags.  Here the shard is cut out of the HOST copy of the
// global graph into one contiguous host buffer (pinned by the caller), so the device never holds
// the global graph: per phase the two shards of the partition's chunk pair are copied in
// (grappa_shard_load, async) and the partition is extracted on the device from them
// (grappa_repartition_shards).  Device memory is then O(two chunks + one partition), whatever
// the graph size.
//
// Image layout (every array 256-byte aligned after a 256-byte header):
//   header {magic, chunk, feat_dim, dtype, n_rows, nnz}
//   ids int32[n] | rowptr int64[n+1] (from 0) | col int32[nnz] | labels int32[n] | train u8[n] |
//   x [n x feat_dim] (fp32, or bf16 rounded to nearest even like the device's conversion)
#include <cstring>
#include <thread>
#include <vector>

#include "part.cuh"

namespace grappa {

static constexpr uint64_t kShardMagic = 0x6472616873707267ull;   // "grpshard"

struct ShardImgHdr {
    uint64_t magic;
    int32_t chunk, feat_dim;
    int32_t dtype, pad;
    int64_t n_rows, nnz;
};

static size_t al256h(size_t b) { return (b + 255) / 256 * 256; }

struct ShardImgLayout {
    size_t ids, rowptr, col, labels, train, x, total;
};
static ShardImgLayout img_layout(int64_t n, int64_t nnz, int32_t feat_dim, grappa_dtype dtype) {
    const size_t esz = dtype == GRAPPA_BF16 ? 2 : 4;
    ShardImgLayout L;
    size_t o = 256;
    L.ids = o; o += al256h((size_t)n * 4);
    L.rowptr = o; o += al256h((size_t)(n + 1) * 8);
    L.col = o; o += al256h((size_t)(nnz > 0 ? nnz : 0) * 4);
    L.labels = o; o += al256h((size_t)n * 4);
    L.train = o; o += al256h((size_t)n);
    L.x = o; o += al256h((size_t)n * feat_dim * esz);
    L.total = o;
    return L;
}

// fp32 -> bf16, round to nearest even (finite inputs; NaN kept quiet), as __float2bfloat16_rn
static inline uint16_t bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

template <class F>
static void parallel_for(int64_t n, int threads, F f) {
    if (threads <= 1 || n < 4096) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        const int64_t a = t * per, b = std::min(n, a + per);
        if (a >= b) break;
        th.emplace_back([=] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

}  // namespace grappa

using namespace grappa;

extern "C" grappa_status grappa_shard_image_size(const int64_t* rowptr, int64_t num_nodes, const int32_t* chunk_of,
                                                 int32_t chunk, int32_t feat_dim, grappa_dtype dtype,
                                                 int64_t* n_rows, int64_t* nnz, size_t* bytes) {
    GRAPPA_ARG(rowptr && chunk_of && bytes, GRAPPA_E_ARG, "grappa_shard_image_size: null argument");
    GRAPPA_ARG(num_nodes > 0 && num_nodes < (1ll << 31), GRAPPA_E_ARG, "grappa_shard_image_size: N out of range");
    GRAPPA_ARG(feat_dim >= 0 && feat_dim % 16 == 0, GRAPPA_E_SHAPE,
               "grappa_shard_image_size: feat_dim must be a multiple of 16");
    int64_t n = 0, m = 0;
    for (int64_t v = 0; v < num_nodes; v++)
        if (chunk_of[v] == chunk) {
            n++;
            m += rowptr[v + 1] - rowptr[v];
        }
    GRAPPA_ARG(n > 0, GRAPPA_E_EMPTY, "grappa_shard_image_size: chunk %d is empty", chunk);
    if (n_rows) *n_rows = n;
    if (nnz) *nnz = m;
    *bytes = img_layout(n, m, feat_dim, dtype).total;
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_shard_image_build(const int64_t* rowptr, const int32_t* col, int64_t num_nodes,
                                                  const float* feats, int32_t feat_dim, grappa_dtype dtype,
                                                  const int32_t* chunk_of, int32_t chunk, const uint8_t* train_mask,
                                                  const int32_t* labels, void* image, size_t image_bytes,
                                                  int32_t threads) {
    GRAPPA_ARG(rowptr && col && chunk_of && train_mask && image, GRAPPA_E_ARG,
               "grappa_shard_image_build: null argument");
    GRAPPA_ARG(feat_dim == 0 || feats, GRAPPA_E_ARG, "grappa_shard_image_build: feat_dim > 0 without features");
    int64_t n = 0, m = 0;
    size_t need = 0;
    GRAPPA_TRY(grappa_shard_image_size(rowptr, num_nodes, chunk_of, chunk, feat_dim, dtype, &n, &m, &need));
    GRAPPA_ARG(image_bytes >= need, GRAPPA_E_ARG, "grappa_shard_image_build: image of %zu bytes, need %zu",
               image_bytes, need);
    const ShardImgLayout L = img_layout(n, m, feat_dim, dtype);
    char* base = (char*)image;
    ShardImgHdr h{kShardMagic, chunk, feat_dim, (int32_t)dtype, 0, n, m};
    memset(base, 0, 256);
    memcpy(base, &h, sizeof(h));
    int32_t* ids = (int32_t*)(base + L.ids);
    int64_t* rp = (int64_t*)(base + L.rowptr);
    int32_t* cl = (int32_t*)(base + L.col);
    int32_t* lab = (int32_t*)(base + L.labels);
    uint8_t* tr = (uint8_t*)(base + L.train);
    // rows in ascending global id, their shard rowptr (sequential: a prefix sum)
    int64_t i = 0, e = 0;
    rp[0] = 0;
    for (int64_t v = 0; v < num_nodes; v++)
        if (chunk_of[v] == chunk) {
            ids[i] = (int32_t)v;
            e += rowptr[v + 1] - rowptr[v];
            rp[++i] = e;
        }
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    // adjacency, labels, train flags, features: rows copied in parallel
    parallel_for(n, threads, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; r++) {
            const int64_t v = ids[r];
            const int64_t d = rowptr[v + 1] - rowptr[v];
            if (d) memcpy(cl + rp[r], col + rowptr[v], (size_t)d * 4);
            lab[r] = labels ? labels[v] : 0;
            tr[r] = train_mask[v];
            if (feat_dim) {
                const float* src = feats + (size_t)v * feat_dim;
                if (dtype == GRAPPA_BF16) {
                    uint16_t* dst = (uint16_t*)(base + L.x) + (size_t)r * feat_dim;
                    for (int32_t f = 0; f < feat_dim; f++) dst[f] = bf16_rne(src[f]);
                } else {
                    memcpy((float*)(base + L.x) + (size_t)r * feat_dim, src, (size_t)feat_dim * 4);
                }
            }
        }
    });
    return GRAPPA_OK;
}

extern "C" grappa_status grappa_shard_load(grappa_ctx* ctx, const void* image, grappa_shard** inout, void* stream) {
    CallScope call_scope(ctx, stream);
    GRAPPA_ARG(ctx && image && inout, GRAPPA_E_ARG, "grappa_shard_load: null argument");
    ShardImgHdr h;
    memcpy(&h, image, sizeof(h));
    GRAPPA_ARG(h.magic == kShardMagic && h.n_rows > 0 && h.nnz >= 0, GRAPPA_E_ARG,
               "grappa_shard_load: not a shard image");
    const grappa_dtype dt = (grappa_dtype)h.dtype;
    const ShardImgLayout L = img_layout(h.n_rows, h.nnz, h.feat_dim, dt);
    const char* base = (const char*)image;
    cudaStream_t s = (cudaStream_t)stream;
    grappa_shard* sh = *inout ? *inout : new grappa_shard();
    auto fail = [&](grappa_status st) {
        if (!*inout) grappa_shard_destroy(sh);
        return st;
    };
    const int64_t n = h.n_rows, m = h.nnz;
    const size_t esz = dt == GRAPPA_BF16 ? 2 : 4;
    grappa_status st;
    if ((st = sh->ids.grow((size_t)n * 4)) != GRAPPA_OK || (st = sh->rowptr.grow((size_t)(n + 1) * 8)) != GRAPPA_OK ||
        (st = sh->col.grow((size_t)(m > 0 ? m : 1) * 4)) != GRAPPA_OK || (st = sh->labels.grow((size_t)n * 4)) != GRAPPA_OK ||
        (st = sh->train.grow((size_t)n)) != GRAPPA_OK ||
        (h.feat_dim && (st = sh->x.grow((size_t)n * h.feat_dim * esz)) != GRAPPA_OK))
        return fail(st);
    struct C { void* d; size_t off, bytes; } cp[] = {
        {sh->ids.p, L.ids, (size_t)n * 4}, {sh->rowptr.p, L.rowptr, (size_t)(n + 1) * 8},
        {sh->col.p, L.col, (size_t)m * 4}, {sh->labels.p, L.labels, (size_t)n * 4},
        {sh->train.p, L.train, (size_t)n}, {sh->x.p, L.x, (size_t)n * h.feat_dim * esz}};
    for (const C& c : cp)
        if (c.bytes && cudaMemcpyAsync(c.d, base + c.off, c.bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            set_error("grappa_shard_load: %s", cudaGetErrorString(cudaGetLastError()));
            return fail(GRAPPA_E_CUDA);
        }
    grappa_shard_info& I = sh->info;
    I.chunk = h.chunk; I.n_rows = n; I.nnz = m; I.feat_dim = h.feat_dim; I.dtype = dt;
    I.ids = (const int32_t*)sh->ids.p; I.rowptr = (const int64_t*)sh->rowptr.p; I.col = (const int32_t*)sh->col.p;
    I.x = h.feat_dim ? sh->x.p : nullptr; I.labels = (const int32_t*)sh->labels.p;
    I.train = (const uint8_t*)sh->train.p;
    *inout = sh;
    return GRAPPA_OK;
}
