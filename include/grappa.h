/*
 * grappa.h -- C ABI of libgrappa.so, the B200 (sm_100a) hot path of Grappa's
 * partition-isolated, gradient-only GNN training step (arXiv 2602.01872).
 *
 * Citations: P:<n> = PAPER.md line n (section / equation / algorithm named beside it),
 * S:<n> = SPEC.md line n, R<k> = reading k in DESIGN.md §2 (where the paper is silent).
 *
 * Conventions (all entry points)
 *  - Plain C types only.  "dev" pointers are CUDA device pointers, "host" pointers are
 *    host memory.  Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Tensors passed in are CALLER-OWNED; the library never frees them.  grappa_ctx,
 *    grappa_part, grappa_shard and grappa_batch are LIBRARY-OWNED and released by their
 *    *_destroy call.
 *  - Dense node tensors are row-major [rows x cols] with cols = the padded width given in
 *    the call (every width is a multiple of 16; padded columns must be zero on input and
 *    are kept zero on output).  Weights are fp32 row-major [f_in x f_out].
 *  - Every call enqueues on the given stream and returns without a device sync, except
 *    grappa_partition, grappa_repartition(_ex/_shards), grappa_shard_extract,
 *    grappa_shard_exchange, grappa_part_query and grappa_check (documented).
 *  - Argument errors are detected synchronously before anything is enqueued and return a
 *    status != GRAPPA_OK; grappa_last_error() then returns a thread-local message.  After
 *    an error the outputs are unspecified and nothing leaks.  One host thread per ctx.
 *  - Determinism: results are bitwise reproducible run to run for fixed inputs, device
 *    count and dtype (no floating-point atomics; fixed-order split-K and reductions).
 */
#ifndef GRAPPA_H
#define GRAPPA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GRAPPA_OK = 0,
    GRAPPA_E_ARG = 1,        /* invalid argument value (e.g. C<2, base==swept)            */
    GRAPPA_E_SHAPE = 2,      /* dimension mismatch / width not a multiple of 16          */
    GRAPPA_E_EMPTY = 3,      /* empty seed set                      */
    GRAPPA_E_NONFINITE = 4,  /* non-finite gradient or coverage factor     */
    GRAPPA_E_SUPPORT = 5,    /* reserved: q = 0 in the node-level variant         */
    GRAPPA_E_NOMEM = 6,      /* device allocation failed                                  */
    GRAPPA_E_CUDA = 7,       /* CUDA runtime error                                        */
    GRAPPA_E_NCCL = 8        /* NCCL error                                                */
} grappa_status;

typedef enum { GRAPPA_F32 = 0, GRAPPA_BF16 = 1 } grappa_dtype;
/* GRAPPA_GAT (reading R35): one attention head over N_loc(v) + v,
 * e_vu = LeakyReLU_0.2(z_u . a_src + z_v . a_dst), alpha = row softmax, out_v = sum alpha_vu z_u,
 * z = h W; weights per layer [W; a_src; a_dst] = fp32 [(f_in + 2) x f_out] (W rows first). */
typedef enum { GRAPPA_GCN = 0, GRAPPA_SAGE = 1, GRAPPA_GAT = 2 } grappa_arch;

/* Coverage-correction factor kinds (§3.4):
 *  NONE           c = 1                         (ablation "UW")
 *  UNIFORM        eq:correction_uniform P:303-305, the minimum-distance factor (Thm 2)
 *  RESAMPLING     eq:resampling P:344-346 literal, with SPEC guards D<eps -> 1, cap c_max
 *                 (S:351); the paper's deployed factor
 *  RESAMPLING_HM  reading R13 (not the default): sum s_v / sum s_v d_g/d_l
 *  NODE           node-level estimator (eq. (4)/(9) P:249-289, reading R30): the
 *                 correction lives inside the gradient (layer calls with
 *                 GRAPPA_LAYER_NODE_LEVEL, per-target weights d_l/d_g); the batch factor is 1 */
typedef enum {
    GRAPPA_CORR_NONE = 0,
    GRAPPA_CORR_UNIFORM = 1,
    GRAPPA_CORR_RESAMPLING = 2,
    GRAPPA_CORR_RESAMPLING_HM = 3,
    GRAPPA_CORR_NODE = 4
} grappa_corr;

typedef struct grappa_ctx grappa_ctx;    /* per process + GPU: NCCL comm, workspaces      */
typedef struct grappa_part grappa_part;  /* per partition: local CSR, maps, degrees, seeds */

/* Global graph in CSR (undirected, symmetric, sorted, deduplicated, no self loops;
 * S:22-28).  Device pointers, caller-owned. */
typedef struct {
    int64_t num_nodes;
    int64_t nnz;
    const int64_t* rowptr;   /* dev [num_nodes+1] */
    const int32_t* col;      /* dev [nnz]         */
} grappa_csr;

/* Read-only view of a partition (all pointers dev, owned by the grappa_part). */
typedef struct {
    int64_t n_core;             /* local nodes = rows of the local CSR: |base| + |swept|
                                   core nodes, then n_halo halo nodes (halo-1 mode)     */
    int64_t nnz;                /* local directed edges (cut edges dropped)             */
    int64_t n_seeds;            /* core train nodes (reading R3)                 */
    int32_t base, swept;        /* chunk ids                                            */
    int32_t feat_dim;           /* padded feature width of x                            */
    grappa_dtype dtype;         /* storage dtype of x                                   */
    const int64_t* rowptr;      /* [n_core+1] local CSR                                 */
    const int32_t* col;         /* [nnz] local ids, ascending per row (R14)             */
    const int32_t* core_global; /* [n_core] global id of local id i (ascending)         */
    const int32_t* d_l;         /* [n_core] local degree                                */
    const int32_t* d_g;         /* [n_core] global degree                               */
    const float* norm_gcn;      /* [n_core] (d_l+1)^-1/2  (GCN, virtual self loop, R5)  */
    const float* norm_sage;     /* [n_core] 1/d_l, 0 where d_l = 0 (SAGE mean, R6)      */
    const int32_t* seeds;       /* [n_seeds] local ids, ascending                       */
    const int32_t* labels;      /* [n_core]                                             */
    const void* x;              /* [n_core x feat_dim] core features, local order       */
    int64_t n_heavy;            /* rows split into segments for the SpMM (d_l > seg)    */
    int64_t n_slots;            /* partial-sum slots used by split rows                 */
    /* coverage statistics over the seeds (full-graph mode: s_v = d_l)                  */
    double c_uniform;           /* eq:correction_uniform                                */
    double c_resampling;        /* eq:resampling with guards (eps 1e-9, c_max 10)       */
    double c_resampling_hm;     /* reading R13                                          */
    int64_t D;                  /* sum_{seeds, d_l>0} (d_g - d_l), exact integer        */
    /* node-level estimator weights (eq. (9), R30), three fp32 rows of n_core:
     *   [0, n)   w_v = d_l/d_g (1 where d_g = 0)
     *   [n, 2n)  w_v * norm_gcn[v]        (GCN backward gather scale)
     *   [2n, 3n) w_v * norm_sage[v] = 1/d_g where d_l > 0, else 0 (SAGE mean scale)      */
    const float* node_w;
    /* halo-1 mode (GRAPPA_PART_HALO1, R33): local ids n_core - n_halo .. n_core - 1 are halo
     * nodes (empty rows); the local operator is not symmetric, so the library also keeps its
     * transpose (the backward aggregations run on it).  n_halo = 0 and t_* = NULL otherwise. */
    int64_t n_halo;
    const int64_t* t_rowptr;    /* [n_core+1] transpose CSR (sources of every column)   */
    const int32_t* t_col;       /* [nnz] source local ids, ascending per row            */
} grappa_part_info;

/* ----------------------------------------------------------------------------------- */
const char* grappa_version(void);
/* Thread-local message describing the most recent failure on this thread. */
const char* grappa_last_error(void);

/* NCCL bootstrap: rank 0 fills 128 bytes; the caller broadcasts them (torch.distributed)
 * and passes them to grappa_ctx_create on every rank. */
grappa_status grappa_nccl_unique_id(void* out128 /* host, 128 bytes */);

/* Create a context on `device`.  nccl_uid == NULL or nranks == 1 -> single GPU, no NCCL.
 * Otherwise a collective: every rank must call it with the same uid (ncclCommInitRank).
 * Library-owned device memory is cudaMalloc'd (grappa_ctx_create_ex to supply an allocator). */
grappa_status grappa_ctx_create(int device, const void* nccl_uid, int rank, int nranks,
                                grappa_ctx** out);
/* Caller allocator for the device memory of library-owned objects (partitions, shards, batches,
 * ctx workspaces): alloc(bytes, stream, user) returns a device pointer usable on `stream` (the
 * stream of the API call that grows the buffer; NULL = legacy default) or NULL on failure
 * (-> GRAPPA_E_NOMEM); free(ptr, bytes, stream, user) returns it (stream = the one it was
 * allocated for; the library frees only after its own work on that stream is enqueued, so a
 * stream-ordered pool such as PyTorch's caching allocator may reuse it in stream order).  Buffers
 * grown while the call's stream is being captured into a CUDA graph are cudaMalloc'd instead.
 * Objects keep the allocator they were grown with, so the callbacks must stay valid until every
 * object created through this ctx is destroyed.  alloc == NULL or free == NULL -> cudaMalloc. */
typedef void* (*grappa_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*grappa_free_fn)(void* ptr, size_t bytes, void* stream, void* user);
grappa_status grappa_ctx_create_ex(int device, const void* nccl_uid, int rank, int nranks,
                                   grappa_alloc_fn alloc, grappa_free_fn free_fn, void* alloc_user,
                                   grappa_ctx** out);
void grappa_ctx_destroy(grappa_ctx* ctx);

/* a1 -- random chunking, performed once (§3.3; reading R1):
 *   chunk_of[v] = pi_seed(v) mod C, pi = 4-round Feistel bijection on [0,N), cycle-walked.
 * chunk_of: dev int32[num_nodes] (out).  chunk_sizes: host int64[C] (out; the call syncs
 * the stream).  Errors: E_ARG if C < 2 or C > num_nodes. */
grappa_status grappa_partition(grappa_ctx* ctx, int64_t num_nodes, int32_t num_chunks,
                               uint64_t seed, int32_t* chunk_of, int64_t* chunk_sizes,
                               void* stream);

/* a3 -- super-epoch repartition (§3.3, §4; S:135-143 induced-core mode):
 * extract the partition of chunk pair {base, swept} from the replicated global CSR:
 * core = nodes of both chunks in ascending global id (local id = rank), each core row keeps
 * the neighbours inside the core (cut edges dropped), d_l/d_g, GCN/SAGE norms, core
 * features gathered into local order, labels, seeds = core train nodes, coverage stats.
 *   g         dev global CSR;  feats dev [N x feat_dim] (dtype);  chunk_of dev int32[N];
 *   train_mask dev uint8[N];  labels dev int32[N].
 *   *inout    NULL -> a new grappa_part is created; otherwise its buffers are reused.
 * Syncs the stream (twice: to size outputs and to publish the coverage statistics).
 * Errors: E_ARG base==swept or out of range; E_EMPTY if the partition has no
 * seeds. */
grappa_status grappa_repartition(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                 int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                 int32_t num_chunks, int32_t base, int32_t swept,
                                 const uint8_t* train_mask, const int32_t* labels,
                                 grappa_part** inout, void* stream);
/* grappa_repartition with flags:
 *   GRAPPA_PART_HALO1 : halo-1 partition ("halo nodes ... cache boundary neighbors", P:196
 *     "incorporated as a halo node"; readings R33/R34): halo = non-core neighbours
 *     of core nodes; core rows keep ALL their neighbours (d_l = d_g), halo rows are empty; local
 *     ids = core (ascending global id) then halo (ascending global id); each row lists its
 *     neighbours in ascending global id; features gathered for core and halo rows; seeds = core
 *     train nodes.  One more host sync (halo count) and a transpose (radix sort) are built.
 * flags = 0 is grappa_repartition.  Errors as grappa_repartition; E_ARG for unknown flags. */
#define GRAPPA_PART_HALO1 1u
grappa_status grappa_repartition_ex(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                    int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                    int32_t num_chunks, int32_t base, int32_t swept,
                                    const uint8_t* train_mask, const int32_t* labels, unsigned flags,
                                    grappa_part** inout, void* stream);
/* a3 for every partition of a super-epoch switch in one call (induced-core partitions from the
 * replicated global CSR): partition k = chunk pair {bases[k], swepts[k]} (host int32[n_parts]),
 * written to parts[k] (host array of n_parts grappa_part*; NULL entries -> created, others
 * reused).  Each partition is bitwise the one grappa_repartition builds; the switch costs two host
 * syncs in total (sizes after the counting pass, statistics at the end) instead of five per
 * partition.  chunk_sizes: host int64[num_chunks], grappa_partition's output for this chunk map
 * (core sizes are allocated from it and checked against the device counts).  Other arguments as
 * grappa_repartition.  Errors: as grappa_repartition (E_EMPTY names the seedless pair), E_ARG if
 * chunk_sizes disagree with chunk_of; on error no partition is published and created ones are
 * destroyed. */
grappa_status grappa_repartition_batch(grappa_ctx* ctx, const grappa_csr* g, const void* feats, int32_t feat_dim,
                                       grappa_dtype dtype, const int32_t* chunk_of, int32_t num_chunks,
                                       const int64_t* chunk_sizes, int32_t n_parts, const int32_t* bases,
                                       const int32_t* swepts, const uint8_t* train_mask, const int32_t* labels,
                                       grappa_part** parts, void* stream);
/* Switch index of a (global CSR, chunk map) pair, built once per run (the chunk map is fixed for
 * the whole run, "performed only once") and passed to grappa_repartition_batch_ix:
 *   per-edge chunk bytes ec[e] = chunk_of[col[e]]  (device uint8 [nnz], library-owned) -- the
 *       switch's "is this neighbour in {base, swept}" test becomes a coalesced byte stream;
 *   per-chunk node counts and sums of the nodes' global degrees (host; bound the task tables).
 * grappa_index_create: one kernel pass over the edges and one host sync.  The index refers to
 * g->rowptr, g->col and chunk_of by address: the caller keeps them alive and unchanged while the
 * index is used (grappa_repartition_batch_ix checks the addresses and sizes, not the contents).
 * Errors: E_ARG (C outside [2, 255], N outside int32, null), E_NOMEM, E_CUDA.
 * grappa_index_query copies the per-chunk counts / degree sums into host int64[C] (either NULL). */
typedef struct grappa_index grappa_index;
grappa_status grappa_index_create(grappa_ctx* ctx, const grappa_csr* g, const int32_t* chunk_of,
                                  int32_t num_chunks, grappa_index** out, void* stream);
grappa_status grappa_index_query(const grappa_index* ix, int64_t* chunk_sizes, int64_t* chunk_degrees);
void grappa_index_destroy(grappa_index* ix);
/* grappa_repartition_batch with a prebuilt index (chunk map and C taken from it): the same
 * partitions, bitwise.  grappa_repartition_batch itself builds a temporary index per call. */
grappa_status grappa_repartition_batch_ix(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                          int32_t feat_dim, grappa_dtype dtype, const grappa_index* ix,
                                          const int64_t* chunk_sizes, int32_t n_parts, const int32_t* bases,
                                          const int32_t* swepts, const uint8_t* train_mask,
                                          const int32_t* labels, grappa_part** parts, void* stream);
grappa_status grappa_part_query(const grappa_part* part, grappa_part_info* out);
void grappa_part_destroy(grappa_part* part);

/* ---- sharded mode (a3 (i); "each chunk stored ... loaded" , §4 "at a switch,
 * workers load the new chunk's edges", "the only data moved ... at super-epoch switches";
 * SURVEY §8e per-super-epoch shift permutation).  Instead of replicating the global graph on
 * every GPU, each rank keeps only the CHUNK SHARDS it owns -- the rows of one chunk: its nodes
 * in ascending global id, their full adjacency lists (global neighbour ids, sorted), features,
 * labels and train flags -- and at a super-epoch switch receives the swept chunk's shard from
 * its owner (NCCL point-to-point over NVLink).  The partition is then built from the two shards
 * (grappa_repartition_shards); it is bitwise the partition grappa_repartition builds from the
 * replicated graph.  Only induced-core partitions (halo-1 needs non-core features). */
typedef struct grappa_shard grappa_shard;   /* library-owned; grappa_shard_destroy */
typedef struct {
    int32_t chunk;              /* chunk id c                                           */
    int32_t feat_dim;           /* padded feature width (0 = no features)               */
    grappa_dtype dtype;         /* storage dtype of x                                   */
    int64_t n_rows;             /* |chunk c|                                            */
    int64_t nnz;                /* sum of the rows' global degrees                      */
    const int32_t* ids;         /* dev [n_rows] global ids, ascending                  */
    const int64_t* rowptr;      /* dev [n_rows+1], rowptr[0] = 0                        */
    const int32_t* col;         /* dev [nnz] global neighbour ids, ascending per row    */
    const void* x;              /* dev [n_rows x feat_dim]                              */
    const int32_t* labels;      /* dev [n_rows]                                         */
    const uint8_t* train;       /* dev [n_rows]                                         */
} grappa_shard_info;
/* Cut chunk `chunk`'s shard out of a global CSR (the loader step a rank runs once for every
 * chunk it owns; the global graph may be dropped afterwards).  Inputs as grappa_repartition.
 * *inout NULL -> new shard, else its buffers are reused.  Syncs the stream once (row count).
 * Errors: E_ARG chunk out of range / null; E_EMPTY if the chunk has no nodes. */
grappa_status grappa_shard_extract(grappa_ctx* ctx, const grappa_csr* g, const void* feats,
                                   int32_t feat_dim, grappa_dtype dtype, const int32_t* chunk_of,
                                   int32_t num_chunks, int32_t chunk, const uint8_t* train_mask,
                                   const int32_t* labels, grappa_shard** inout, void* stream);
grappa_status grappa_shard_query(const grappa_shard* shard, grappa_shard_info* out);
void grappa_shard_destroy(grappa_shard* shard);
/* One point-to-point transfer of a shard: exactly one of send / recv is non-NULL. */
typedef struct {
    int32_t peer;               /* the other rank (may be this rank: a self copy through NCCL) */
    const grappa_shard* send;   /* send this shard to peer                              */
    grappa_shard** recv;        /* receive a shard from peer into *recv (NULL -> created) */
} grappa_shard_xfer;
/* Collective over the ctx's NCCL communicator (ctx created with a uid, any nranks >= 1):
 * every transfer listed on one rank must be matched by the opposite transfer on its peer, and
 * transfers between the same two ranks must be listed in the same order on both.  Three grouped
 * NCCL rounds: a 32-byte header per transfer (then one host sync to size the receive buffers),
 * an 8-byte status from every receiver to its sender (one more host sync: both sides of every
 * transfer agree that the receiver could allocate before any array moves, so a failure on one
 * rank is reported on its peers instead of leaving them in an unmatched send), then the arrays
 * (ids, rowptr, col, x, labels, train; counted in grappa_comm_bytes' `other`).  Errors: E_ARG
 * no communicator / bad peer / both or neither of send, recv / malformed header; E_NOMEM;
 * E_NCCL (also on a sender whose receiver failed). */
grappa_status grappa_shard_exchange(grappa_ctx* ctx, int32_t n_xfers, const grappa_shard_xfer* xfers,
                                    void* stream);
/* a3 from two shards: the partition of chunk pair {base->chunk, swept->chunk} (rank table from
 * the replicated chunk map, 4 bytes per node; rows, features, labels and train flags from the
 * shards).  Output, syncs and errors as grappa_repartition (E_ARG if the shards hold the same
 * chunk, their feature widths or dtypes differ, or a chunk id is out of range). */
grappa_status grappa_repartition_shards(grappa_ctx* ctx, const grappa_shard* base, const grappa_shard* swept,
                                        const int32_t* chunk_of, int64_t num_nodes, int32_t num_chunks,
                                        grappa_part** inout, void* stream);

/* a3 from two shards with flags: 0 is grappa_repartition_shards; GRAPPA_PART_HALO1 builds the
 * halo-1 partition (R33/R34) whose core part is complete but whose halo rows (features, global
 * degree, label, node weight) are PENDING: they live in other chunks' shards and arrive with
 * grappa_halo_exchange (layer calls reject a pending partition with E_ARG). */
grappa_status grappa_repartition_shards_ex(grappa_ctx* ctx, const grappa_shard* base, const grappa_shard* swept,
                                           const int32_t* chunk_of, int64_t num_nodes, int32_t num_chunks,
                                           unsigned flags, grappa_part** inout, void* stream);
/* Halo feature all-to-all of sharded halo-1 partitions ("Halo node features are pre-cached at
 * super-epoch boundaries", "synchronize halo features", "Feature gathering during
 * repartitioning uses all-to-all collectives").  COLLECTIVE over the ctx's communicator: every rank
 * calls it once per partition build, in the same order; part = this rank's pending partition or
 * NULL (a rank without one still answers requests).  shards: the n_shards chunk shards this rank
 * owns (host array of handles); chunk_owner: host int32[C], the rank owning each chunk's shard;
 * chunk_of: dev [N].  Rounds: per-owner request counts (one host sync), an ok word from every rank
 * (both sides agree before any array moves), request ids (int32, ascending per owner), replies
 * (feature row in the storage dtype, global degree, label per request) -- counted in
 * grappa_comm_bytes' `other`.  Afterwards the partition is bitwise the replicated path's halo-1
 * partition.  Errors: E_ARG (no communicator, C > 64, bad owner, a shard this rank does not own,
 * mismatched feature format, a requested node absent from its owner's shards), E_NOMEM, E_NCCL. */
grappa_status grappa_halo_exchange(grappa_ctx* ctx, grappa_part* part, int32_t n_shards,
                                   const grappa_shard* const* shards, const int32_t* chunk_owner,
                                   const int32_t* chunk_of, int32_t num_chunks, void* stream);

/* Host images of chunk shards -- the data loader of capacity mode from chunk shards (§8f row 3:
 * Alg. 1 with M < P beyond HBM; "trades training time for memory capacity" P:395;
 * partitions in CPU memory loaded onto the GPU P:410; RMAT-36 one partition at a time P:656).
 * A shard image is one contiguous HOST buffer (caller-owned; pin it for asynchronous loads) with a
 * 256-byte header and the arrays of grappa_shard_info (ids, rowptr from 0, global col, labels,
 * train flags, x in the storage dtype), cut out of a HOST copy of the global graph, so the
 * device never holds the global graph: per phase the two shards of the partition's chunk pair are
 * loaded (grappa_shard_load) and the partition extracted from them (grappa_repartition_shards),
 * bitwise the partition grappa_repartition builds.
 *   grappa_shard_image_size   host rowptr [N+1], chunk map [N]: rows / edges of chunk `chunk` and
 *                             the image size in bytes.  E_EMPTY for an empty chunk.
 *   grappa_shard_image_build  write chunk `chunk`'s image (host fp32 feats [N x feat_dim], cast to
 *                             dtype: bf16 rounds to nearest even; labels may be NULL; `threads` <=
 *                             0 -> all host cores).  E_ARG if image_bytes is too small.
 *   grappa_shard_load         (re)allocate *inout (NULL -> new shard) and enqueue the H2D copies of
 *                             an image on stream; no host sync (the header is read on the host);
 *                             the image must stay valid until the copies complete. */
grappa_status grappa_shard_image_size(const int64_t* rowptr, int64_t num_nodes, const int32_t* chunk_of,
                                      int32_t chunk, int32_t feat_dim, grappa_dtype dtype, int64_t* n_rows,
                                      int64_t* nnz, size_t* bytes);
grappa_status grappa_shard_image_build(const int64_t* rowptr, const int32_t* col, int64_t num_nodes,
                                       const float* feats, int32_t feat_dim, grappa_dtype dtype,
                                       const int32_t* chunk_of, int32_t chunk, const uint8_t* train_mask,
                                       const int32_t* labels, void* image, size_t image_bytes, int32_t threads);
grappa_status grappa_shard_load(grappa_ctx* ctx, const void* image, grappa_shard** inout, void* stream);

/* Host-memory image of a partition's arrays (sizes as in grappa_part_info; any field may be
 * NULL = not transferred).  Used when partitions live in host memory between phases -- the
 * paper keeps partitions in CPU memory and loads them to the GPU; the bench's
 * end-to-end number streams them per phase.  Host buffers should be pinned for overlap. */
typedef struct {
    int64_t* rowptr;        /* [n_core+1] */
    int32_t* col;           /* [nnz]      */
    int32_t* d_l;           /* [n_core]   */
    float* norm_gcn;        /* [n_core]   */
    float* norm_sage;       /* [n_core]   */
    int32_t* seeds;         /* [n_seeds]  */
    int32_t* labels;        /* [n_core]   */
    void* x;                /* [n_core x feat_dim] */
    float* node_w;          /* [3 x n_core] (grappa_part_info.node_w) */
} grappa_part_host;
/* device -> host copy of the selected arrays (enqueued on stream) */
grappa_status grappa_part_download(const grappa_part* part, const grappa_part_host* dst, void* stream);
/* host -> device copy into the partition's own buffers (enqueued on stream; same sizes).
 * The image must be this partition's own (as written by grappa_part_download): the SpMM
 * metadata derived at repartition time (split rows, degree-bucketed row order) is kept. */
grappa_status grappa_part_upload(grappa_part* part, const grappa_part_host* src, void* stream);

/* Partition images: the whole partition (arrays, SpMM plans, transpose) serialised into ONE
 * host buffer, for phase-parallel capacity mode -- partitions parked in host memory and streamed
 * to a GPU slot per phase (Alg. 1 with M < P; "trades training time for memory
 * capacity" P:395; partitions in CPU memory, loaded to the GPU).
 *   grappa_part_image_bytes  size of the image of `part` (0 if part is NULL)
 *   grappa_part_save         enqueue D2H copies of every array into host (pinned for overlap)
 *                            and write the header at once; the image is complete when the
 *                            stream reaches this point.  E_ARG if host_bytes is too small.
 *   grappa_part_image_info   the image's grappa_part_info (pointers NULL), read on the host
 *   grappa_part_load         (re)allocate *inout's buffers (growing only) and enqueue H2D copies
 *                            of an image; *inout NULL -> a new part.  No host sync: the header is
 *                            read from host memory.  The image must stay valid until the copies
 *                            are done (stream order).  E_ARG if host is not an image. */
size_t grappa_part_image_bytes(const grappa_part* part);
grappa_status grappa_part_save(const grappa_part* part, void* host, size_t host_bytes, void* stream);
grappa_status grappa_part_image_info(const void* host, grappa_part_info* out);
grappa_status grappa_part_load(grappa_part** inout, const void* host, void* stream);

/* Workspace sizes (bytes) for one layer call on `part`; `saved` persists fwd -> bwd. */
size_t grappa_layer_saved_bytes(const grappa_part* part, grappa_arch arch, int32_t f_in,
                                int32_t f_out, grappa_dtype dtype);
size_t grappa_layer_ws_bytes(const grappa_part* part, grappa_arch arch, int32_t f_in,
                             int32_t f_out, grappa_dtype dtype);

/* a4 -- one isolated message-passing layer, forward (§3.2; §5.1):
 *   GCN  (R5):  h_out = act( Ahat h_in W ),  Ahat = Dt^-1/2 (A_loc + I) Dt^-1/2,
 *                      Dt = d_l + 1; computed transform-first: T' = N h_in W (tensor-core
 *                      GEMM, row scale n_v = Dt^-1/2 in its epilogue), then
 *                      h_out_v = act(n_v (T'_v + sum_{u in N_loc(v)} T'_u)) (SpMM).
 *                      `saved` unused (may be NULL).
 *   SAGE (R6):  M = D_l^-1 A_loc h_in (SpMM, zero rows where d_l = 0, kept in
 *                      `saved`), h_out = act([h_in | M] [W_self; W_nbr]) (one GEMM, K = 2 f_in).
 *   GAT  (R35):        [z | s t] = h_in [W | W a_src | W a_dst] (one GEMM; z, s, t kept in
 *                      `saved` with the attention coefficients), alpha per edge and self loop
 *                      (row log-sum-exp), h_out = act(sum_u alpha_vu z_u) (the SpMM with
 *                      per-edge weights).  f_out <= 256 (bf16) / 128 (fp32), else E_SHAPE.
 *   act = ReLU if relu != 0 else identity (output layer).
 *   h_in dev [n_core x f_in], h_out dev [n_core x f_out] (dtype); w dev fp32: GCN
 *   [f_in x f_out], SAGE [2 f_in x f_out] (W_self rows first).  ws: grappa_layer_ws_bytes.
 * Errors: E_SHAPE if f_in or f_out is not a positive multiple of 16. */
grappa_status grappa_layer_fwd(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                               int32_t f_in, int32_t f_out, int relu, const void* h_in,
                               const float* w, void* h_out, void* saved, void* ws,
                               grappa_dtype dtype, void* stream);

/* Layer flags (grappa_layer_fwd_ex / grappa_layer_bwd_ex / grappa_minibatch_step_ex):
 *   GRAPPA_LAYER_NODE_LEVEL : node-level estimator (eq. (4)/(9) P:249-289; R30) --
 *     every target's aggregated neighbour message is multiplied by w_v = d_l/d_g:
 *       GCN  Ahat_w = N (diag(w) A_loc + I) N   (self term unweighted)
 *       SAGE M = diag(w) D_l^-1 A_loc h_in       (= local sum / d_g)
 *     and the backward is the exact transpose (Ahat_w^T = N (A_loc diag(w) + I) N); GCN
 *     evaluates it from dz' = w dz rounded to the storage dtype (reading R30c), so the gather
 *     is unweighted (ws: grappa_layer_ws_bytes holds dz').
 *     Pair it with GRAPPA_CORR_NODE in the aggregation (batch factor 1).               */
#define GRAPPA_LAYER_NODE_LEVEL 4u
/*   GRAPPA_LAYER_INPUT : the model's first layer (its backward is called with dz_in = NULL).
 *     GCN then evaluates aggregate-first, Z = (Ahat h_in) W: the forward keeps P = Ahat h_in in
 *     `saved` (size: grappa_layer_saved_bytes_ex with this flag), and the backward is dW = P^T dz
 *     alone -- no aggregation (a re-association of the same products, reading R29; one bf16
 *     rounding of P instead of one of h_in W).  P is formed as N (h'_v + sum_u h'_u) from the
 *     pre-scaled rows h' = N h_in (rounded to the storage dtype; reading R29c), so the gather
 *     carries no per-edge weight.  The backward takes no normalised-gradient flags.
 *     No effect for SAGE / GAT (SAGE is aggregate-first already). */
#define GRAPPA_LAYER_INPUT 8u
size_t grappa_layer_saved_bytes_ex(const grappa_part* part, grappa_arch arch, int32_t f_in,
                                   int32_t f_out, grappa_dtype dtype, unsigned flags);
/* grappa_layer_fwd with flags (0 = grappa_layer_fwd).  Errors: E_ARG for unknown flags. */
grappa_status grappa_layer_fwd_ex(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                  int32_t f_in, int32_t f_out, int relu, const void* h_in,
                                  const float* w, void* h_out, void* saved, void* ws,
                                  grappa_dtype dtype, unsigned flags, void* stream);

/* a6 -- the layer's backward (exact reverse mode; ReLU'(0) = 0, R16):
 *   dz_out   dev [n_core x f_out]: dL/dZ of THIS layer's pre-activation output.
 *   dw       dev fp32, same shape as w: dL/dW, combined over row splits in fixed order.
 *   dz_in    dev [n_core x f_in] or NULL (first layer: skipped): dL/dZ of the previous
 *            layer's pre-activation, i.e. (dL/dh_in) * 1[h_in > 0] when relu_in != 0.
 *   GCN : dT = Ahat dz_out (SpMM; Ahat symmetric because the induced subgraph of an
 *         undirected graph is symmetric), dW = h_in^T dT, dh_in = dT W^T.
 *   SAGE: [dW_self; dW_nbr] = [h_in | M]^T dz_out, dh_in = dz_out W_self^T
 *         + A_loc D_l^-1 (dz_out W_nbr^T).                                              */
grappa_status grappa_layer_bwd(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                               int32_t f_in, int32_t f_out, int relu_in, const void* dz_out,
                               const void* h_in, const float* w, const void* saved, float* dw,
                               void* dz_in, void* ws, grappa_dtype dtype, void* stream);

/* grappa_layer_bwd with normalised-gradient flags (GCN only; reading R29).  With
 * N = diag(norm_gcn), Ahat dz = N (A_loc + I) (N dz): a caller that chains GCN layers can pass
 * gradients pre-multiplied by N, so every backward aggregation gathers unweighted rows.
 *   GRAPPA_BWD_DZ_OUT_NORMED : dz_out holds N dz_out.
 *   GRAPPA_BWD_DZ_IN_NORMED  : dz_in receives N dz_in (the relu' gate is applied as usual).
 * dw is the same in every mode.  flags = 0 is grappa_layer_bwd.  GRAPPA_LAYER_NODE_LEVEL (any
 * arch) backpropagates through the node-level operator of grappa_layer_fwd_ex.  Errors: E_ARG
 * for unknown flags or a normalised-gradient flag with arch SAGE. */
#define GRAPPA_BWD_DZ_OUT_NORMED 1u
#define GRAPPA_BWD_DZ_IN_NORMED 2u
grappa_status grappa_layer_bwd_ex(grappa_ctx* ctx, const grappa_part* part, grappa_arch arch,
                                  int32_t f_in, int32_t f_out, int relu_in, const void* dz_out,
                                  const void* h_in, const float* w, const void* saved, float* dw,
                                  void* dz_in, void* ws, grappa_dtype dtype, unsigned flags,
                                  void* stream);

/* a5 -- mean softmax cross-entropy over the partition's seeds (R8):
 *   L = (1/#S) sum_{v in S} [logsumexp(Z_v[0:K]) - Z_v[y_v]];  dZ_v = (softmax - e_y)/#S on
 *   seeds, 0 on every other row and on padded columns K..k_pad-1 (masked to -inf).
 *   logits/dlogits dev [n_core x k_pad] (dtype); loss_dev dev float64[1] (out).
 * Errors: E_ARG if num_classes > k_pad; E_EMPTY if the partition has no seeds. */
grappa_status grappa_loss(grappa_ctx* ctx, const grappa_part* part, const void* logits,
                          int32_t num_classes, int32_t k_pad, void* dlogits, double* loss_dev,
                          grappa_dtype dtype, void* stream);
/* with flags: GRAPPA_LOSS_DZ_NORMED writes N dZ (rows times norm_gcn, the GCN
 * normalised-gradient chain of reading R29), for a last GCN layer's backward called with
 * GRAPPA_BWD_DZ_OUT_NORMED.  The loss value is unchanged.  flags = 0 is grappa_loss. */
#define GRAPPA_LOSS_DZ_NORMED 1u
grappa_status grappa_loss_ex(grappa_ctx* ctx, const grappa_part* part, const void* logits,
                             int32_t num_classes, int32_t k_pad, void* dlogits, double* loss_dev,
                             grappa_dtype dtype, unsigned flags, void* stream);

/* a7 + a8 -- coverage-corrected aggregation and optimizer step (P:291-306 eq:batch-estimator,
 * Alg. 1, "applied immediately before the all-reduce"):
 *   comm <- (c_p / m_active) * grad, cast to comm_dtype (one fused scale/cast pass that also
 *   flags non-finite values), then ncclAllReduce(sum) of comm across the context's ranks
 *   =>  grad = (1/M) sum_p c_p g_p (R9; fp32, or rounded to bf16 once and summed in bf16 by
 *   NCCL when comm_dtype = GRAPPA_BF16), then, if lr != 0, theta <- theta - lr * grad (SGD,
 *   S:429-437, R10).  The update is skipped on the device when the aggregated gradient -- or any
 *   aggregated since the last grappa_check -- is non-finite ("non-finite grad -> error"):
 *   theta is never written with a non-finite step, and grappa_check reports E_NONFINITE.
 *   part == NULL marks a rank with no active partition in this phase (contributes zeros).
 *   c_p is the factor of kind `corr` from the partition's coverage statistics
 *   (grappa_part_info): UNIFORM c_uniform; RESAMPLING from the exact integer D:
 *   1 if D < eps, else min(1/D, c_max) (SPEC CorrectionConfig S:311-314 --
 *   eps > 0, c_max >= 1; the oracle's defaults are 1e-9 and 10); RESAMPLING_HM c_resampling_hm;
 *   1 for NONE and NODE (node-level: the correction is in the gradient).
 *   grad, theta: dev fp32 [n_params].  A COLLECTIVE when the ctx has >1 rank.
 *   Errors: E_ARG (null, m_active < 1, eps <= 0, c_max < 1, unknown corr / comm_dtype, lr != 0
 *   without theta); E_NONFINITE if c_p is not finite; E_NOMEM (bf16 comm buffer);
 *   E_NCCL. */
grappa_status grappa_aggregate_grads(grappa_ctx* ctx, const grappa_part* part, grappa_corr corr,
                                     double eps, double c_max, float* grad, int64_t n_params,
                                     int32_t m_active, grappa_dtype comm_dtype, float lr, float* theta,
                                     void* stream);

/* a7 with an explicit factor (mini-batch mode: c_p is the batch's factor, grappa_batch_factors).
 * Same semantics as grappa_aggregate_grads with c_p = c (c = 0 for an idle rank). */
grappa_status grappa_aggregate_grads_c(grappa_ctx* ctx, double c, float* grad, int64_t n_params,
                                       int32_t m_active, grappa_dtype comm_dtype, float lr, float* theta,
                                       void* stream);

/* Bytes this ctx has moved between GPUs since creation, by purpose (host counters, updated when
 * a call enqueues the transfer): grad = gradient all-reduce payloads (per rank, the buffer
 * size of every ncclAllReduce), other = everything else (shard / halo exchange at super-epoch
 * switches).  The paper's invariant "cross-server traffic consists only of gradient all-reduce"
 * is that `other` does not grow inside training iterations. */
grappa_status grappa_comm_bytes(const grappa_ctx* ctx, int64_t* grad_bytes, int64_t* other_bytes);

/* ---------------------------------------------------------------- a10: mini-batch mode
 * Isolated mini-batch sampling (config 4): P:139/P:177 (§3.2 sampling mode, k-hop subgraphs
 * from the local partition only), P:382 (Alg. 1 isolated_sampling), P:489 (B = 1000,
 * fanouts {15,10,5}).  Readings R23-R28:
 *   epoch order  seeds sorted by (h(seed, epoch, gid), gid)
 *   hop h        each target v keeps min(f_h, d_l(v)) distinct local neighbours, uniform
 *                without replacement, drawn by Floyd's algorithm over neighbour positions
 *                (R24; keys h(h(seed, epoch, batch, h), gid(v), j))
 *   fanouts      each in [1, 32] (P:489's {15,10,5}, {25,10}, {20,15,10,5})
 *   replay       grappa_sample_async replays the batch's launch sequence as a CUDA graph from
 *                the second call with the same (partition, n_batch, fanouts) on a non-default
 *                stream (per-call values through pinned memory); results are identical
 *   sources      targets (prefix, same order) then new nodes in ascending local id
 *   fanouts      listed input -> output layer: hop 1 (the seeds) uses fanouts[L-1]
 * GraphSAGE only (config 4 is SAGE-3). */
typedef struct grappa_batch grappa_batch;   /* library-owned layered blocks of one batch */

typedef struct {
    int32_t n_dst, n_src;       /* targets (rows) / sources (columns) of the block          */
    int64_t nnz;
    const int64_t* rowptr;      /* dev [n_dst+1]  block CSR, col = source positions asc.    */
    const int32_t* col;         /* dev [nnz]                                                */
    const int64_t* t_rowptr;    /* dev [n_src+1]  transpose (source -> target positions)    */
    const int32_t* t_col;       /* dev [nnz]                                                */
    const float* inv_cnt;       /* dev [n_dst]    1/|S(v)|, 0 for an empty sample           */
    const int32_t* src;         /* dev [n_src]    partition-local id of each source         */
    const float* inv_cnt_node;  /* dev [n_dst]    (d_l/d_g)(v) / |S(v)| (node-level, R30)   */
} grappa_block_info;

/* Epoch order of the partition's seeds (R23): order dev int32[n_seeds] (out, local ids). */
grappa_status grappa_epoch_seeds(grappa_ctx* ctx, const grappa_part* part, uint64_t seed,
                                 int64_t epoch, int32_t* order, void* stream);
/* Sample the L blocks of one batch (P:139, P:382 isolated_sampling).  Per target v
 * at hop h: min(f_h, d_l(v)) distinct local neighbours, uniform without replacement, drawn by
 * Floyd's algorithm over neighbour positions keyed by h(h(seed, epoch, batch_index, h), gid v, j)
 * (reading R24); hop 1 uses the LAST fanout (R25); sources = targets then new nodes in ascending
 * local id (R26).  batch: dev int32[n_batch] local seed ids; fanouts: host int32[n_layers]
 * (input -> output, each <= 32).  *inout NULL -> created, else reused.  Syncs once.
 * Errors: E_ARG (n_layers < 1 or > 8, fanout outside [1, 32], n_batch < 1). */
grappa_status grappa_sample(grappa_ctx* ctx, const grappa_part* part, const int32_t* batch,
                            int32_t n_batch, const int32_t* fanouts, int32_t n_layers,
                            uint64_t seed, int64_t epoch, int64_t batch_index,
                            grappa_batch** inout, void* stream);
/* The same call split in two, so a caller can sample batch i+1 on a side stream while batch i
 * trains: grappa_sample_async enqueues every kernel and a D2H copy of the block sizes into
 * pinned memory owned by the batch (no host sync); grappa_sample_wait blocks until that copy
 * has landed and publishes the sizes and coverage factors.  Until then grappa_batch_query /
 * grappa_batch_factors / grappa_minibatch_step return E_ARG and grappa_minibatch_ws_bytes 0.
 * grappa_sample_event returns the cudaEvent_t (as void*) recorded after the sample's last
 * kernel, for a consumer stream to wait on.  Reusing a batch object for a new sample is the
 * caller's to order after every consumer of its previous blocks (stream/event order).
 * grappa_sample = grappa_sample_async + grappa_sample_wait. */
grappa_status grappa_sample_async(grappa_ctx* ctx, const grappa_part* part, const int32_t* batch,
                                  int32_t n_batch, const int32_t* fanouts, int32_t n_layers,
                                  uint64_t seed, int64_t epoch, int64_t batch_index,
                                  grappa_batch** inout, void* stream);
grappa_status grappa_sample_wait(grappa_batch* b);
grappa_status grappa_sample_event(const grappa_batch* b, void** event_out);
/* layer l = 0 (input) .. n_layers-1 (output: its targets are the batch seeds) */
grappa_status grappa_batch_query(const grappa_batch* b, int32_t layer, grappa_block_info* out);
/* Coverage factors of the batch over its seeds with s_v = hop-1 sample size (R28):
 * eq:correction_uniform, eq:resampling (SPEC guards), and the R13 reading. */
grappa_status grappa_batch_factors(const grappa_batch* b, double* c_uniform,
                                   double* c_resampling, double* c_resampling_hm);
void grappa_batch_destroy(grappa_batch* b);

/* One isolated SAGE mini-batch forward + loss + backward on the sampled blocks:
 *   h_0 = x[src of layer 0]; layer l: h_{l+1}[v] = act(h_l[v] W_self + mean_{u in S(v)} h_l[u]
 *   W_nbr); loss = mean softmax-CE over the batch seeds; grad (dev fp32, flat theta layout:
 *   per layer [W_self; W_nbr] blocks of dims_pad[l] x dims_pad[l+1]) <- dL/dtheta.
 *   dims_pad: host int32[n_layers+1] (multiples of 16; dims_pad[0] = the partition's
 *   feat_dim).  ws: ws_bytes >= grappa_minibatch_ws_bytes(b, ...) (E_ARG otherwise: the
 *   workspace depends on the sampled sizes of THIS batch).  hidden_out: NULL, or host array
 *   of n_layers-1 dev pointers receiving h_1..h_{L-1} (rows n_dst of layers 0..L-2). */
size_t grappa_minibatch_ws_bytes(const grappa_batch* b, int32_t n_layers, const int32_t* dims_pad,
                                 grappa_dtype dtype);
grappa_status grappa_minibatch_step(grappa_ctx* ctx, const grappa_part* part, const grappa_batch* b,
                                    int32_t n_layers, const int32_t* dims_pad, int32_t num_classes,
                                    const float* theta, float* grad, void* ws, size_t ws_bytes,
                                    double* loss_dev, void* const* hidden_out, grappa_dtype dtype,
                                    void* stream);
/* The step enqueues a wait on the batch's sample-completion event first, so the batch may have
 * been sampled on another stream (grappa_sample_async).
 * with flags: GRAPPA_LAYER_NODE_LEVEL scales every target's sampled mean by d_l/d_g (R30;
 * inv_cnt_node instead of inv_cnt, forward and backward).  flags = 0 is the call above. */
grappa_status grappa_minibatch_step_ex(grappa_ctx* ctx, const grappa_part* part, const grappa_batch* b,
                                       int32_t n_layers, const int32_t* dims_pad, int32_t num_classes,
                                       const float* theta, float* grad, void* ws, size_t ws_bytes,
                                       double* loss_dev, void* const* hidden_out, grappa_dtype dtype,
                                       unsigned flags, void* stream);

/* Sync the stream and report asynchronous faults: E_NONFINITE if any aggregated gradient
 * since the last check was non-finite, E_CUDA / E_NCCL on device or communicator errors. */
grappa_status grappa_check(grappa_ctx* ctx, void* stream);

/* Number of kernels this ctx has launched (for the bench's gpu_launches claim). */
int64_t grappa_launch_count(const grappa_ctx* ctx);

/* Per-kernel-class timing for the roofline report.  While enabled, every call of a class
 * records a CUDA event pair on its launch stream around that class's launches, plus the
 * call's ALGORITHMIC bytes and flops (DESIGN.md §4 gives the per-unit formulas):
 *   SPMM     per edge 4 (col) + 4 (edge weight, GCN) + w*s (gathered row); per row 8 (rowptr)
 *            + 8 (scales) + w*s (self row, GCN) + w*s (output) [+ w*s accumulate, + w*s mask]
 *   GEMM     (M*K*s + K*N*4 + M*N*s [+ M*N*s mask]) bytes, 2*M*N*K flops
 *   GEMM_TN  (M*K*s + M*N*s + K*N*4) bytes, 2*M*N*K flops (split-K partials excluded)
 * enable(on=1) clears previous records; read() syncs and sums one class. */
typedef enum {
    GRAPPA_K_SPMM = 0,
    GRAPPA_K_GEMM = 1,
    GRAPPA_K_GEMM_TN = 2,
    GRAPPA_K_LOSS = 3,
    GRAPPA_K_AGG = 4,
    GRAPPA_K_REPART = 5,
    GRAPPA_K_SAMPLE = 6,     /* mini-batch sampler (grappa_sample, incl. its one host sync) */
    GRAPPA_K_NCLASS = 7
} grappa_kclass;
/* Test hook (per ctx): select an alternative implementation of the same arithmetic so tests can
 * cross-check kernels against each other.  Every variant computes the documented result.
 *   op "gemm": 0 = tensor cores (tcgen05 for bf16, split-fp32 tcgen05 for fp32; default),
 *              1 = CUDA-core kernels (bf16; 128x128 FFMA tiles for fp32), 2 = small-tile CUDA-core.
 *   op "spmm": 0 = row-group kernel (rows of <= 32 vectors) over the degree-bucketed row order
 *              (default), 1 = warp per row, 2 = row-group with 8 loads in flight, 3 = row-group
 *              over the natural row order, 4 = TMA row gathers into a shared-memory ring (spmm_tma.cu; bf16
 *              unweighted widths 80..128 only, others fall back to 0), 5 = row-group with the
 *              previous per-edge-predicated unweighted schedule (same sums, bitwise).
 *   op "pair": 0 = GCN backward computes dz_in and dW in one pass over dT and h_in (bf16,
 *              default), 1 = the two separate GEMMs.
 *   op "wstream": tcgen05 transform GEMM's weight operand: 0 = converted once into a bf16
 *              image and streamed per k-block when the call has <= 2 row tiles per SM, else
 *              resident in shared memory (default), 1 = always streamed, 2 = resident whenever
 *              it fits.  Same products and fp32 accumulation order either way (bitwise).
 * Returns E_ARG for a null ctx, an unknown op or an out-of-range variant. */
grappa_status grappa_set_kernel_variant(grappa_ctx* ctx, const char* op, int variant);

/* Roofline probes (diagnostics; bench.py's live ceilings).  Allocates its own
 * buffers (cudaMalloc / cudaFree: synchronises the device; never call inside graph capture),
 * runs one warm-up launch and `iters` timed launches on `stream` (CUDA events) and returns the
 * achieved bandwidth in *gbps (1e9 bytes/s):
 *   GRAPPA_PROBE_HBM_COPY    dst = src over `bytes` each (use bytes >> L2): (read + write) / time
 *   GRAPPA_PROBE_L2_READ     8 passes of coalesced 16-byte reads over `bytes` (L2-resident if
 *                            bytes < L2): bytes read / time
 *   GRAPPA_PROBE_L2_GATHER   whole-row gathers of a `bytes`-sized table of row_bytes rows (16 *
 *                            a divisor of 32) at random row ids read from an index array, the
 *                            SpMM's access pattern with no arithmetic: row bytes / time
 * Errors: E_ARG (bytes < 1 MiB or not a multiple of 16, iters < 1, bad row_bytes or kind),
 * E_NOMEM. */
#define GRAPPA_PROBE_HBM_COPY 0
#define GRAPPA_PROBE_L2_READ 1
#define GRAPPA_PROBE_L2_GATHER 2
grappa_status grappa_roofline_probe(grappa_ctx* ctx, int kind, int64_t bytes, int32_t row_bytes, int32_t iters,
                                    double* gbps, void* stream);

grappa_status grappa_profile_enable(grappa_ctx* ctx, int on);
grappa_status grappa_profile_read(grappa_ctx* ctx, int kclass, double* ms, int64_t* calls,
                                  double* bytes, double* flops);

#ifdef __cplusplus
}
#endif
#endif /* GRAPPA_H */
