"""Host-side driver: Algorithm 1 (phase-parallel training) over the grappa C ABI.

PAPER: Alg. 1 P:367-393 (§3.6), super-epochs P:188-190 / P:413, sweep schedule P:207,
batch-level correction before the all-reduce P:306 / P:407.

One process per GPU.  With P partitions (logical workers, W = P = C) and G ranks, each
epoch runs ceil(P/G) phases; in phase i rank r trains partition i*G + r (if it exists) and
all ranks aggregate (NCCL all-reduce inside grappa_aggregate_grads, M = active ranks).
The only cross-GPU traffic inside an iteration is that all-reduce; partitions are
re-extracted on every rank's GPU from the replicated global CSR at super-epoch switches
(no feature exchange needed in replicated mode).

Everything numeric happens in libgrappa.so; this module only schedules calls and owns
buffers (torch CUDA tensors).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import (BF16, BWD_DZ_IN_NORMED, BWD_DZ_OUT_NORMED, F32, LAYER_INPUT, LAYER_NODE_LEVEL, Context, Part,
               Shard, grappa_aggregate_grads, grappa_shard_load, shard_image, grappa_layer_bwd, grappa_layer_bwd_ex, grappa_layer_fwd_ex,
               Index, grappa_loss, grappa_partition, grappa_repartition, grappa_repartition_batch, grappa_repartition_shards,
               grappa_halo_exchange, grappa_shard_exchange, grappa_shard_extract, layer_saved_bytes, layer_ws_bytes)


def sweep_schedule(C: int, W: int):
    """a2 (reading R2 for W < C): per super-epoch t = 1..cycle, the
    (base, swept) chunk pair of each worker."""
    if not (1 <= W <= C and C >= 2):
        raise ValueError("need 1 <= W <= C, C >= 2")
    if W == C:
        return [[(w, (w + t) % C) for w in range(W)] for t in range(1, C)]
    pairs = [(i, j) for i in range(C) for j in range(i + 1, C)]
    cycle = -(-len(pairs) // W)
    return [[pairs[((t - 1) * W + w) % len(pairs)] for w in range(W)] for t in range(1, cycle + 1)]


def merge_step_factors(per_rank) -> list:
    """per_rank[r] = [(partition, coverage, active), ...] for the same lock-step sequence of
    optimizer steps; returns the (partition, coverage) observations in step order, ranks in
    ascending order within a step (idle ranks dropped) -- the controller's input (R32)"""
    out = []
    for k in range(len(per_rank[0]) if per_rank else 0):
        for r in per_rank:
            if r[k][2] > 0:
                out.append((int(r[k][0]), float(r[k][1])))
    return out


def phase_plan(W: int, G: int, rank: int):
    """Alg. 1 with P = W partitions on G ranks (M = G partitions per phase):
    phase i -> (worker i*G + rank, or None if this rank idles in a ragged last phase,
    m_active = number of active partitions in the phase)."""
    nphase = -(-W // G)
    plan = []
    for i in range(nphase):
        w = i * G + rank
        plan.append((i, w if w < W else None, min(G, W - i * G)))
    return plan


def shard_owner(c: int, G: int) -> int:
    """sharded mode: chunk c's shard lives on rank c mod G (with W = C: worker w's base chunk w
    sits on the rank that trains w, phase_plan)"""
    return c % G


def shard_plan(pairs, W: int, G: int):
    """a3 (i) in sharded mode ("workers load the new chunk's edges"): per phase
    i, the point-to-point shard transfers (chunk, src rank, dst rank) that give the worker
    i*G + r on rank r both chunks of its pair.  One global order (phase, dst, chunk) that every
    rank derives identically, so transfers between two ranks are listed in the same order on
    both.  With W = C = G this is the shift permutation: rank r receives chunk (r + t) mod C
    from rank (r + t) mod C and sends its own chunk to rank (r - t) mod C."""
    plan = []
    for i in range(-(-W // G)):
        xs = []
        for r in range(G):
            w = i * G + r
            if w >= W:
                continue
            for c in sorted(set(pairs[w])):
                o = shard_owner(c, G)
                if o != r:
                    xs.append((c, o, r))
        plan.append(xs)
    return plan


def shard_xfers(xs, rank: int):
    """this rank's side of one phase of shard_plan: sends [(dst, chunk)], receives [(src, chunk)],
    each in the plan's global order"""
    return ([(dst, c) for (c, src, dst) in xs if src == rank],
            [(src, c) for (c, src, dst) in xs if dst == rank])


@dataclass
class ModelSpec:
    arch: str            # "gcn" | "sage"
    dims: list           # logical widths [F, hidden..., K]
    dims_pad: list       # padded widths (multiples of 16)

    @property
    def depth(self):
        return len(self.dims) - 1

    def layer_shapes(self):
        """padded weight block shape per layer: GCN [fin, fout]; SAGE [2 fin, fout];
        GAT [fin + 2, fout] (W, then the a_src and a_dst rows)"""
        if self.arch == "gat":
            return [(self.dims_pad[l] + 2, self.dims_pad[l + 1]) for l in range(self.depth)]
        m = 1 if self.arch == "gcn" else 2
        return [(m * self.dims_pad[l], self.dims_pad[l + 1]) for l in range(self.depth)]

    def n_params(self):
        return sum(a * b for a, b in self.layer_shapes())


class Trainer:
    """Partition-isolated full-graph training (Alg. 1) on this rank's GPU."""

    def __init__(self, ctx: Context, rowptr, col, x, labels, train_mask, spec: ModelSpec, weights,
                 num_chunks: int, chunk_seed: int, corr: str = "resampling", lr: float = 0.003,
                 repartition_every: int = 10, dtype: str = "f32", num_workers: int | None = None,
                 stream=None, controller=None, halo: bool = False, capacity: bool = False,
                 sharded: bool = False, comm_dtype: str = "f32", eps: float = 1e-9, c_max: float = 10.0):
        self.ctx = ctx
        self.dev = torch.device("cuda", ctx.device)
        self.stream = stream or torch.cuda.current_stream(self.dev)
        self.spec = spec
        self.C = num_chunks
        self.W = num_workers or num_chunks                     # P = W logical workers
        self.G = ctx.nranks
        self.rank = ctx.rank
        self.corr = corr
        self.lr = lr
        # a7 arguments: all-reduce payload dtype (fused scale/cast) and the R12 guards
        self.comm_dtype, self.eps, self.c_max = comm_dtype, eps, c_max
        self.rep_every = repartition_every
        # optional §3.5 controller (paper_2602_01872_b200.controller.Controller): decides the
        # super-epoch switches instead of the fixed `repartition_every`
        self.controller = controller
        self.halo = halo                 # halo-1 partitions (R33) instead of induced-core
        # capacity mode (Alg. 1 with M < P beyond HBM): partitions live as images in
        # pinned host memory and are streamed into one of two device slots per phase
        # capacity="shards": the global graph never reaches the device -- every chunk's shard is
        # an image in pinned host memory, and each phase loads its pair's two shards and extracts
        # the partition from them on the device (device memory O(two chunks + one partition))
        self.capacity = capacity
        self.cap_shards = capacity == "shards"
        if capacity not in (False, True, "shards"):
            raise ValueError("capacity must be False, True (partition images) or 'shards' (chunk-shard images)")
        # sharded mode (a3 (i)): keep only the owned chunk shards, exchange swept shards at switches
        self.sharded = sharded
        if sharded and capacity:
            raise ValueError("sharded mode holds its partitions in HBM (no capacity mode)")
        if self.cap_shards and halo:
            raise ValueError("capacity mode from chunk shards builds induced-core partitions")
        self.host_imgs: dict = {}
        self.img_bytes: dict = {}
        self.cap_slots = None
        self.t_ctrl = 1
        self._steps = []
        self.dt = BF16 if dtype == "bf16" else F32
        self.tdt = torch.bfloat16 if self.dt == BF16 else torch.float32
        self.schedule = sweep_schedule(self.C, self.W)
        as_t = lambda a, dt: (a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))).to(self.dev, dt)
        if self.cap_shards:
            self._init_shard_images(ctx, rowptr, col, x, labels, train_mask, chunk_seed)
            self._init_params(spec, weights)
            return
        # replicated global graph + node data, resident in HBM for the whole run
        self.rowptr = as_t(rowptr, torch.int64)
        self.col = as_t(col, torch.int32)
        self.N = self.rowptr.numel() - 1
        # features: cast to the storage dtype on the host first (papers-scale fp32 features
        # are 57 GB; bf16 halves both the host->device copy and the transient device copy)
        xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        self.x = xt.to(self.tdt).to(self.dev).contiguous()
        self.labels = as_t(labels, torch.int32)
        self.train = as_t(train_mask, torch.uint8)
        # a1: chunk map, once
        self.chunk_of = torch.empty(self.N, dtype=torch.int32, device=self.dev)
        self.chunk_sizes = grappa_partition(ctx, self.N, self.C, chunk_seed, self.chunk_of, self.stream)
        self.nnz_global = int(self.col.numel())
        if sharded:
            # cut this rank's chunk shards out, then drop the replicated graph: from here on the
            # rank holds its shards, the chunk map and the partitions it trains
            self.shards = {c: grappa_shard_extract(ctx, self.rowptr, self.col, self.x, self.dt, self.chunk_of,
                                                   self.C, c, self.train, self.labels, None, self.stream)
                           for c in range(self.C) if shard_owner(c, self.G) == self.rank}
            self.recv_slots = [Shard(), Shard()]
            self.owners = [shard_owner(c, self.G) for c in range(self.C)]
            self.rowptr = self.col = self.x = self.labels = self.train = None
        self._init_params(spec, weights)

    def _init_shard_images(self, ctx, rowptr, col, x, labels, train_mask, chunk_seed):
        """capacity mode from chunk shards: the chunk map on the device (a1), every chunk's shard
        cut out of the HOST graph into a pinned image (grappa_shard_image_build); no global array
        is copied to the device"""
        host = lambda a, dt: (a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)).astype(dt, copy=False)
        rowptr, col = host(rowptr, np.int64), host(col, np.int32)
        self.N = rowptr.size - 1
        self.nnz_global = int(col.size)
        self.chunk_of = torch.empty(self.N, dtype=torch.int32, device=self.dev)
        self.chunk_sizes = grappa_partition(ctx, self.N, self.C, chunk_seed, self.chunk_of, self.stream)
        cmap = self.chunk_of.cpu().numpy()
        xf = host(x, np.float32)
        self.shard_imgs = [shard_image(rowptr, col, xf, self.dt, cmap, c, host(train_mask, np.uint8),
                                       host(labels, np.int32)) for c in range(self.C)]
        self.shard_img_bytes = sum(int(im.numel()) for im in self.shard_imgs)
        self.rowptr = self.col = self.x = self.labels = self.train = None
        self.sh_slots = [[Shard(), Shard()], [Shard(), Shard()]]
        self.cap_part = Part()
        self.cap_stream = torch.cuda.Stream(self.dev)

    def _init_params(self, spec, weights):
        # theta / grad: one flat fp32 buffer each -> one all-reduce per iteration
        shapes = spec.layer_shapes()
        self.theta = torch.zeros(spec.n_params(), dtype=torch.float32, device=self.dev)
        self.grad = torch.zeros_like(self.theta)
        self.w_views, self.dw_views, off = [], [], 0
        for (a, b) in shapes:
            self.w_views.append(self.theta[off:off + a * b].view(a, b))
            self.dw_views.append(self.grad[off:off + a * b].view(a, b))
            off += a * b
        for l, ws in enumerate(weights):
            blk = np.concatenate([np.asarray(w, dtype=np.float32) for w in ws], axis=0)
            self.w_views[l].copy_(torch.from_numpy(blk))
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.graph = None                # CUDA graph of one epoch (run_epoch_graph), per super-epoch
        # test instrumentation: phase_probe(phase, worker) is called after every phase step of
        # run_epoch_graph, on the stream the step ran on (inside the capture, so stream-ordered
        # copies it enqueues are replayed with the graph); None in normal runs
        self.phase_probe = None
        self.parts: dict = {}            # worker id -> Part (this rank's workers)
        self.t = None
        self.epoch = 0
        self.losses = []

    def check(self):
        """grappa_check on the training stream: E_NONFINITE if any aggregated gradient since the
        last check was non-finite (its SGD step was skipped on the device), E_CUDA / E_NCCL."""
        self.ctx.check(self.stream)

    # ------------------------------------------------------------------ partitions
    def my_workers(self):
        """workers this rank runs, one per phase: phase i -> worker i*G + rank (>= W: idle)"""
        return [(i, i * self.G + self.rank) for i, _, _ in phase_plan(self.W, self.G, self.rank)]

    def repartition(self, t: int):
        """a3 for super-epoch t on every worker this rank owns.  Drops any captured
        epoch graph first: it holds the previous partitions' sizes, SpMM plans, tensor maps,
        coverage factors and buffer pointers, so it must never be replayed on the new layout."""
        self.graph = None
        self.next_graph = None
        if self.t is not None:
            # the switch synchronises anyway: surface a non-finite aggregate of the last
            # super-epoch now (the device skipped those updates)
            self.check()
        pairs = self.schedule[(t - 1) % len(self.schedule)]
        if self.cap_shards:              # partitions are extracted per phase (_run_epoch_shards)
            self.pairs = pairs
            self.t = t
            return None
        if self.capacity:
            return self._repartition_to_host(t, pairs)
        if self.sharded:
            return self._repartition_sharded(t, pairs)
        mine = [w for _, w in self.my_workers() if w < self.W]
        if self.halo:
            for w in mine:
                b, s = pairs[w]
                self.parts[w] = grappa_repartition(self.ctx, self.rowptr, self.col, self.x, self.dt,
                                                   self.chunk_of, self.C, b, s, self.train, self.labels,
                                                   self.parts.get(w), self.stream, halo=True)
        elif mine:
            # every partition of this rank in one call: two host syncs per switch
            # the switch index (per-edge chunk bytes of this graph under the run's chunk map) is
            # built at the first switch and kept: graph and chunk map never change within a run
            if getattr(self, "index", None) is None:
                self.index = Index(self.ctx, self.rowptr, self.col, self.chunk_of, self.C, self.stream)
            got = grappa_repartition_batch(self.ctx, self.rowptr, self.col, self.x, self.dt, self.chunk_of, self.C,
                                           [pairs[w] for w in mine], self.train, self.labels,
                                           [self.parts.get(w) for w in mine], self.stream,
                                           chunk_sizes=self.chunk_sizes, index=self.index)
            self.parts.update(zip(mine, got))
        self.t = t
        self._alloc()

    def _repartition_sharded(self, t, pairs):
        """sharded mode: per phase, the NCCL shard transfers of shard_plan (collective over the
        ranks that take part), then the partition from the two shards; the receive slots are
        reused phase to phase (stream order: a phase's partition is built before the next
        phase's transfers overwrite them)"""
        plan = shard_plan(pairs, self.W, self.G)
        for i, w in self.my_workers():
            snd, rcv = shard_xfers(plan[i], self.rank)
            sends = [(dst, self.shards[c]) for dst, c in snd]
            recvs = [(src, self.recv_slots[k]) for k, (src, c) in enumerate(rcv)]
            got = {c: self.recv_slots[k] for k, (src, c) in enumerate(rcv)}
            if sends or recvs:
                grappa_shard_exchange(self.ctx, sends, recvs, self.stream)
            if w >= self.W:
                if self.halo:            # collective: an idle rank still answers halo requests
                    grappa_halo_exchange(self.ctx, None, list(self.shards.values()), self.owners, self.chunk_of,
                                         self.C, self.stream)
                continue
            b, s = pairs[w]
            sb = self.shards.get(b) or got[b]
            ss = self.shards.get(s) or got[s]
            self.parts[w] = grappa_repartition_shards(self.ctx, sb, ss, self.chunk_of, self.C, self.parts.get(w),
                                                      self.stream, halo=self.halo)
            if self.halo:
                # halo-1 (R33): the halo rows' features, degrees and labels from their chunks'
                # owners -- the all-to-all of P:416, at the switch only
                grappa_halo_exchange(self.ctx, self.parts[w], list(self.shards.values()), self.owners,
                                     self.chunk_of, self.C, self.stream)
        self.t = t
        self._alloc()

    def _repartition_to_host(self, t, pairs):
        """capacity mode: extract each partition into device slot 0, save its image to pinned
        host memory (grappa_part_save), keep only the images"""
        if self.cap_slots is None:
            self.cap_slots = [Part(), Part()]
            self.cap_stream = torch.cuda.Stream(self.dev)
        self.parts = {}
        sizes = []
        for _, w in self.my_workers():
            if w >= self.W:
                continue
            b, s = pairs[w]
            p = grappa_repartition(self.ctx, self.rowptr, self.col, self.x, self.dt, self.chunk_of, self.C,
                                   b, s, self.train, self.labels, self.cap_slots[0], self.stream,
                                   halo=self.halo)
            nb = p.image_bytes()
            host = self.host_imgs.get(w)
            if host is None or host.numel() < nb:
                host = torch.empty(nb + nb // 8, dtype=torch.uint8, pin_memory=True)
                self.host_imgs[w] = host
            p.save(host, self.stream)
            self.img_bytes[w] = nb
            sizes.append(self._sizes(p))
            self.stream.synchronize()              # the image is complete before slot 0 is reused
        self.t = t
        self._alloc(sizes)

    def _sizes(self, p):
        sp = self.spec
        ws = [layer_ws_bytes(p, sp.arch, sp.dims_pad[l], sp.dims_pad[l + 1], self.dt) for l in range(sp.depth)]
        sv = [layer_saved_bytes(p, sp.arch, sp.dims_pad[l], sp.dims_pad[l + 1], self.dt, self._input_flag(l))
              for l in range(sp.depth)]
        return p.n_core, ws, sv

    def _input_flag(self, l: int) -> int:
        """GCN input layer: aggregate-first (GRAPPA_LAYER_INPUT), so its backward needs no
        aggregation (R29 re-association)"""
        return LAYER_INPUT if (l == 0 and self.spec.arch == "gcn") else 0

    def _alloc(self, sizes=None):
        """Activation / workspace buffers sized for the largest partition this rank owns;
        kept across super-epochs (12.5 % headroom) so a switch does not reallocate.
        sizes: [(n_core, ws per layer, saved per layer)] (default: from the resident parts)."""
        sp = self.spec
        if sizes is None:
            sizes = [self._sizes(p) for p in self.parts.values()]
        n_max = max([1] + [z[0] for z in sizes])
        changed = False
        if getattr(self, "_n_cap", 0) < n_max:
            changed = True
            self._n_cap = n_cap = n_max + n_max // 8
            self.H = [None] + [torch.empty(n_cap, sp.dims_pad[l], dtype=self.tdt, device=self.dev)
                               for l in range(1, sp.depth + 1)]
            wmax = max(sp.dims_pad)
            self.dz = [torch.empty(n_cap * wmax, dtype=self.tdt, device=self.dev) for _ in range(2)]
        ws = 1
        saved = []
        for l in range(sp.depth):
            ws = max([ws] + [z[1][l] for z in sizes])
            sb = max([0] + [z[2][l] for z in sizes])
            old = self.saved[l] if getattr(self, "saved", None) else None
            if sb and (old is None or old.numel() < sb):
                old = torch.empty(sb + sb // 8, dtype=torch.uint8, device=self.dev)
                changed = True
            saved.append(old if sb else None)
        if getattr(self, "ws", None) is None or self.ws.numel() < ws:
            self.ws = torch.empty(ws + ws // 8, dtype=torch.uint8, device=self.dev)
            changed = True
        self.saved = saved
        if changed:
            # a captured epoch holds the old buffers' pointers: never replay it on the new ones
            # (the prefetch path reallocates after its last replay was launched and installs
            # the freshly recorded graph at the switch)
            self.graph = None

    # ------------------------------------------------------------------ one iteration
    def forward_backward(self, part: Part):
        """a4-a6 on one isolated partition: L x layer_fwd, loss, L x layer_bwd -> self.grad"""
        sp, n, s = self.spec, part.n_core, self.stream
        L = sp.depth
        dp = sp.dims_pad
        H = [part.x] + [h[:n] for h in self.H[1:]]
        # node-level estimator (corr "node", eq. (9), R30): weighted aggregation in every layer
        nl = LAYER_NODE_LEVEL if self.corr == "node" else 0
        for l in range(L):
            grappa_layer_fwd_ex(self.ctx, part, sp.arch, dp[l], dp[l + 1], l < L - 1, H[l],
                                self.w_views[l], H[l + 1], self.saved[l], self.ws, self.dt,
                                nl | self._input_flag(l), s)
        dz = self.dz[0][: n * dp[L]].view(n, dp[L])
        gcn = sp.arch == "gcn"
        # GCN: the loss writes N dZ directly when the last layer is not the (aggregate-first)
        # input layer, so its backward gathers unweighted rows too (R29)
        last_normed = gcn and L > 1
        grappa_loss(self.ctx, part, H[L], sp.dims[L], dp[L], dz, self.loss_dev, self.dt, s,
                    flags=1 if last_normed else 0)
        for l in range(L - 1, -1, -1):
            dz_in = self.dz[(L - l) % 2][: n * dp[l]].view(n, dp[l]) if l > 0 else None
            # GCN: gradients between layers travel pre-multiplied by N = diag(norm_gcn), so
            # every backward aggregation gathers unweighted rows (grappa_layer_bwd_ex, R29)
            # (the aggregate-first input layer takes its dz un-normalised: no IN_NORMED into l = 0)
            flags = nl | self._input_flag(l)
            if gcn:
                flags |= (BWD_DZ_OUT_NORMED if l > 0 else 0) | (BWD_DZ_IN_NORMED if l > 1 else 0)
            grappa_layer_bwd_ex(self.ctx, part, sp.arch, dp[l], dp[l + 1], l > 0, dz, H[l],
                                self.w_views[l], self.saved[l], self.dw_views[l], dz_in, self.ws,
                                self.dt, flags, s)
            dz = dz_in
        return H[L]

    def phase_step(self, phase: int, worker: int, m_active: int, lr=None):
        part = self.parts.get(worker) if worker < self.W else None
        if part is not None:
            self.forward_backward(part)
        else:
            self.grad.zero_()
        grappa_aggregate_grads(self.ctx, part, self.corr, self.grad, m_active,
                               self.lr if lr is None else lr, self.theta, self.stream, eps=self.eps,
                               c_max=self.c_max, comm_dtype=self.comm_dtype)
        self._steps.append((float(worker), part.info.c_uniform, 1.0) if part is not None
                           else (0.0, 0.0, 0.0))

    # ------------------------------------------------------------------ super-epochs
    def super_epoch(self) -> int:
        """super-epoch index of the next epoch: fixed length, or the controller's count"""
        return self.t_ctrl if self.controller is not None else 1 + self.epoch // self.rep_every

    def end_epoch(self):
        """epoch boundary: feed the controller this epoch's per-step (partition, coverage)
        records of every active rank (gathered, so identical on every rank) and advance the
        super-epoch if it says so (§3.5, R32)"""
        self.epoch += 1
        steps, self._steps = self._steps, []
        if self.controller is None:
            return
        if self.G > 1:
            import torch.distributed as dist
            mine = torch.tensor(steps, dtype=torch.float64, device=self.dev).reshape(-1, 3)
            every = [torch.empty_like(mine) for _ in range(self.G)]
            dist.all_gather(every, mine)
            seq = merge_step_factors([e.cpu().tolist() for e in every])
        else:
            seq = merge_step_factors([steps])
        for p, c in seq:
            self.controller.observe(p, c)
        if self.controller.end_epoch():
            self.t_ctrl += 1

    def run_epoch(self, on_phase=None):
        """One epoch of Alg. 1: ceil(W/G) phases, one aggregate + SGD step per phase."""
        t = self.super_epoch()
        if t != self.t:
            self.repartition(t)
        if self.cap_shards:
            return self._run_epoch_shards(on_phase)
        if self.capacity:
            return self._run_epoch_capacity(on_phase)
        for i, w in self.my_workers():
            m_active = min(self.G, self.W - i * self.G)
            self.phase_step(i, w, m_active)
            if on_phase is not None:
                on_phase()
        self.end_epoch()

    def _run_epoch_capacity(self, on_phase=None):
        """capacity mode: phase k's partition image is copied H2D into slot k % 2 on a copy
        stream while phase k-1 computes on the other slot (grappa_part_load)"""
        plan = self.my_workers()
        free = [None, None]                       # compute done with the slot's previous image

        def load(k):
            _, w = plan[k]
            if w >= self.W:
                return None
            if free[k % 2] is not None:
                self.cap_stream.wait_event(free[k % 2])
            self.cap_slots[k % 2].load_image(self.host_imgs[w], self.cap_stream)
            ev = torch.cuda.Event()
            ev.record(self.cap_stream)
            return ev

        self.cap_stream.wait_stream(self.stream)  # e.g. the repartition's use of slot 0
        ready = load(0) if plan else None
        for k, (i, w) in enumerate(plan):
            nxt = load(k + 1) if k + 1 < len(plan) else None
            if ready is not None:
                self.stream.wait_event(ready)
                self.parts = {w: self.cap_slots[k % 2]}
            else:
                self.parts = {}
            m_active = min(self.G, self.W - i * self.G)
            self.phase_step(i, w, m_active)
            free[k % 2] = torch.cuda.Event()
            free[k % 2].record(self.stream)
            if on_phase is not None:
                on_phase()
            ready = nxt
        self.end_epoch()

    def _run_epoch_shards(self, on_phase=None):
        """capacity mode from chunk shards: phase k's two shard images are copied H2D into shard
        slot k % 2 on a copy stream while phase k-1 computes; the phase then extracts its
        partition from them on the device (grappa_repartition_shards: bitwise the resident
        partition) into the single partition slot and trains on it"""
        plan = self.my_workers()
        extracted = [None, None]                  # slot's previous shards consumed by their extraction

        def load(k):
            _, w = plan[k]
            if w >= self.W:
                return None
            if extracted[k % 2] is not None:
                self.cap_stream.wait_event(extracted[k % 2])
            b, s_ = self.pairs[w]
            A, B = self.sh_slots[k % 2]
            grappa_shard_load(self.ctx, self.shard_imgs[b], A, self.cap_stream)
            grappa_shard_load(self.ctx, self.shard_imgs[s_], B, self.cap_stream)
            ev = torch.cuda.Event()
            ev.record(self.cap_stream)
            return ev

        self.cap_stream.wait_stream(self.stream)
        ready = load(0) if plan else None
        for k, (i, w) in enumerate(plan):
            nxt = load(k + 1) if k + 1 < len(plan) else None
            if ready is not None:
                self.stream.wait_event(ready)
                A, B = self.sh_slots[k % 2]
                part = grappa_repartition_shards(self.ctx, A, B, self.chunk_of, self.C, self.cap_part, self.stream)
                extracted[k % 2] = torch.cuda.Event()
                extracted[k % 2].record(self.stream)
                self.parts = {w: part}
                self._alloc([self._sizes(part)])
            else:
                self.parts = {}
            m_active = min(self.G, self.W - i * self.G)
            self.phase_step(i, w, m_active)
            if on_phase is not None:
                on_phase()
            ready = nxt
        self.end_epoch()

    def run_epoch_graph(self):
        """Same epoch, replayed from a CUDA graph captured once per super-epoch (the phase loop
        issues ~535 launches per products epoch; replay removes the host launch gaps).  On large
        partitions the first epoch of a super-epoch runs eagerly on the main stream while the same
        launches are recorded on a capture stream, so the GPU works through that epoch while the
        host records (capturing alone would leave the GPU idle for the recording +
        instantiation); on small ones (host-bound epochs) it is recorded only, then replayed.

        Prefetched switch (fixed-period super-epochs, replicated induced-core partitions): while
        the GPU replays the LAST epoch of a super-epoch, the host extracts the next super-epoch's
        partitions into the second partition set on a side stream and records their epoch graph;
        the next epoch then only swaps the sets and replays.  The switch's host work (its syncs,
        the ~535 recorded launches) overlaps the GPU instead of pacing it."""
        import os
        import time
        tm = os.environ.get("GRAPPA_GRAPH_TIMING") == "1"     # diagnostic host timings (stderr)
        h0 = time.perf_counter()
        t = self.super_epoch()
        if t != self.t:
            nxt = getattr(self, "next_graph", None)
            if nxt is not None and nxt["t"] == t:
                self._swap_in(nxt)
            else:
                self.repartition(t)                 # drops the previous super-epoch's graph
        h1 = time.perf_counter()
        if getattr(self, "graph", None) is not None:
            self.graph.replay()
            if self.controller is not None:    # the captured steps' factors (fixed per super-epoch)
                self._steps = list(self.graph_steps)
            self._maybe_prefetch(tm)
            self.end_epoch()
            return
        # small partitions (host-bound epochs): record only, then replay -- running the epoch
        # eagerly as well would double the host work that bounds them
        # multi-rank: record only (each communicator then sees one stream of collectives: the
        # captured all-reduces replay in the same order on every rank)
        eager = (self.G == 1 and
                 sum(p.nnz for p in self.parts.values()) >= getattr(self, "graph_eager_min_nnz", 4_000_000))
        g, n_cap, cap_steps, grad_b, h2 = self._capture(eager)
        h3 = time.perf_counter()
        if tm:
            import sys
            print(f"[graph] repartition {1e3 * (h1 - h0):.1f} ms, record{' + eager' if eager else ''} "
                  f"{1e3 * (h2 - h1):.1f} ms, capture_end {1e3 * (h3 - h2):.1f} ms", file=sys.stderr)
        self.graph = g
        self.graph_launches = n_cap
        self.graph_grad_bytes = grad_b       # all-reduce payload bytes per replay (comm counters)
        self.graph_steps = cap_steps
        if not eager:
            g.replay()
            self._steps += cap_steps
        self._maybe_prefetch(tm)
        self.end_epoch()

    def _capture(self, eager: bool):
        """record one epoch of the current self.parts into a CUDA graph (and run it eagerly on the
        main stream at the same time if `eager`); returns (graph, launches, step factors, grad bytes,
        host time at the end of the recording)"""
        import time
        g = torch.cuda.CUDAGraph()
        main = self.stream
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(main)
        n_cap, cap_steps, grad_b = 0, [], 0
        # capture_begin/end directly: torch.cuda.graph() would also run gc.collect() and
        # empty_cache(); relaxed mode lets the eager launches proceed during the capture
        with torch.cuda.stream(cap):
            g.capture_begin(capture_error_mode="relaxed")
            try:
                for i, w in self.my_workers():
                    m_active = min(self.G, self.W - i * self.G)
                    if eager:
                        with torch.cuda.stream(main):
                            self.stream = main
                            self.phase_step(i, w, m_active)       # runs now
                            if self.phase_probe is not None:
                                self.phase_probe(i, w)
                    saved, self._steps = self._steps, []
                    l0 = self.ctx.launches()
                    b0 = self.ctx.comm_bytes()[0]
                    self.stream = cap
                    self.phase_step(i, w, m_active)               # recorded for the replays
                    n_cap += self.ctx.launches() - l0
                    grad_b += self.ctx.comm_bytes()[0] - b0
                    if self.phase_probe is not None:              # its copies are captured too
                        self.phase_probe(i, w)
                    cap_steps += self._steps
                    self._steps = saved
                h2 = time.perf_counter()
            finally:
                self.stream = main
                g.capture_end()
        return g, n_cap, cap_steps, grad_b, h2

    def _prefetch_ok(self) -> bool:
        # one rank only: recording a graph with NCCL all-reduces while the previous graph's
        # all-reduces run on the same communicator has not been exercised on multi-GPU hardware
        return (getattr(self, "prefetch_switch", True) and self.controller is None and not self.halo
                and not self.capacity and not self.sharded and self.rep_every >= 1 and self.G == 1)

    def _maybe_prefetch(self, tm=False):
        """after launching the replay of the last epoch of a super-epoch: build the next one's
        partitions into the other set on a side stream and record their graph (see
        run_epoch_graph)"""
        import time
        if not self._prefetch_ok():
            return
        t1 = 1 + (self.epoch + 1) // self.rep_every
        if t1 == self.t or (getattr(self, "next_graph", None) or {}).get("t") == t1:
            return
        h0 = time.perf_counter()
        nparts = self.build_next_parts(t1)
        h1 = time.perf_counter()
        # buffers for both sets (the running graph's tensors stay valid: any reallocation is
        # stream-ordered after it on the main stream), then record the next epoch on the new set
        self._alloc([self._sizes(p) for p in list(self.parts.values()) + list(nparts.values())])
        self.stream.wait_stream(self.pf_stream)            # the new partitions before their graph
        cur = self.parts
        self.parts = nparts
        try:
            g, n_cap, cap_steps, grad_b, _ = self._capture(eager=False)
        finally:
            self.parts = cur
        self.next_graph = dict(t=t1, parts=nparts, graph=g, launches=n_cap, steps=cap_steps, grad_bytes=grad_b)
        if tm:
            import sys
            print(f"[graph] prefetch of super-epoch {t1}: repartition {1e3 * (h1 - h0):.1f} ms, record "
                  f"{1e3 * (time.perf_counter() - h1):.1f} ms (overlapping the replay)", file=sys.stderr)

    def warm_prefetch(self):
        """pay the prefetched switch's one-time costs before a timed region: the second partition
        set's buffers, the switch index (grappa_index), the prefetch stream and the library's
        side streams at its priority.  Extracts the next super-epoch's partitions into the second
        set once (kept as that set's buffers for the real prefetch) and sizes the activation
        buffers for both sets; call it before the epoch graph is captured.  Without it the first
        prefetch -- 0.1-1 s of host time in first-touch allocations -- fell inside the timed
        epochs."""
        if not self._prefetch_ok():
            return
        nparts = self.build_next_parts(self.t + 1)
        self.pf_stream.synchronize()
        self.alt_parts = dict(nparts)
        self._alloc([self._sizes(p) for p in list(self.parts.values()) + list(nparts.values())])

    def build_next_parts(self, t1: int) -> dict:
        """the partitions of super-epoch t1 in the second partition set, extracted on the side
        stream `pf_stream` (concurrently with work on the main stream); returns worker -> Part"""
        mine = [w for _, w in self.my_workers() if w < self.W]
        pairs = self.schedule[(t1 - 1) % len(self.schedule)]
        if getattr(self, "pf_stream", None) is None:
            # high priority: the switch's kernels are scheduled ahead of the replay they
            # overlap, so the host's size syncs return after the switch's own GPU work
            import os
            self.pf_stream = torch.cuda.Stream(self.dev, priority=int(os.environ.get("GRAPPA_PF_PRIORITY", "-1")))
            self.alt_parts = {}
        if getattr(self, "alt_free", None) is not None:
            self.pf_stream.wait_event(self.alt_free)      # the other set's last graph has finished
        if getattr(self, "index", None) is None:
            self.index = Index(self.ctx, self.rowptr, self.col, self.chunk_of, self.C, self.stream)
        got = grappa_repartition_batch(self.ctx, self.rowptr, self.col, self.x, self.dt, self.chunk_of, self.C,
                                       [pairs[w] for w in mine], self.train, self.labels,
                                       [self.alt_parts.get(w) for w in mine], self.pf_stream,
                                       chunk_sizes=self.chunk_sizes, index=self.index)
        return dict(zip(mine, got))

    def _swap_in(self, nxt):
        """switch to the prefetched super-epoch: its partitions and graph become current; the
        previous set is reused by the next prefetch once its last replay is done"""
        self.check()             # surface a non-finite aggregate of the last super-epoch
        self.alt_parts, self.parts = self.parts, nxt["parts"]
        self.alt_free = torch.cuda.Event()
        self.alt_free.record(self.stream)
        self.graph = nxt["graph"]
        self.graph_launches = nxt["launches"]
        self.graph_grad_bytes = nxt["grad_bytes"]
        self.graph_steps = nxt["steps"]
        self.t = nxt["t"]
        self.next_graph = None

    @property
    def nnz(self):
        return self.nnz_global


class MinibatchTrainer(Trainer):
    """Isolated mini-batch training (sampling mode, config 4).

    Per phase the active workers iterate in lock step over their epoch batches (S:441, S:492:
    a worker with fewer batches cycles its own); every iteration samples the batch's blocks
    inside the partition (grappa_sample), runs one SAGE forward/loss/backward on them
    (grappa_minibatch_step), scales by the batch's coverage factor and all-reduces
    (grappa_aggregate_grads_c) before the SGD step (Alg. 1)."""

    def __init__(self, *args, fanouts=(15, 10, 5), batch_size=1000, sample_seed=0, depth: int = 4, **kw):
        super().__init__(*args, **kw)
        if self.capacity:
            raise ValueError("capacity mode is implemented for full-graph training")
        self.depth = max(1, depth)         # batches sampled ahead (side streams)
        if self.spec.arch != "sage":
            raise ValueError("mini-batch mode is implemented for GraphSAGE (config 4)")
        self.fanouts = list(fanouts)
        self.B = batch_size
        self.sample_seed = sample_seed
        self.batch = None
        self.mb_ws = None
        self.order = None

    def iterations(self, part):
        return 0 if part is None else -(-part.n_seeds // self.B)

    def phase_iterations(self, part):
        n = self.iterations(part)
        if self.G > 1:
            import torch.distributed as dist
            t = torch.tensor([n], dtype=torch.int64, device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            n = int(t.item())
        return n

    def minibatch(self, part, order, it: int, nb: int):
        """sample + forward/backward of batch (it mod nb) -> self.grad; returns the batch
        (unpipelined single-batch path, used by tests and diagnostics)."""
        from . import grappa_sample
        b = it % nb
        seeds = order[b * self.B: min((b + 1) * self.B, order.numel())]
        self.batch = grappa_sample(self.ctx, part, seeds, self.fanouts, self.sample_seed, self.epoch, b,
                                   self.batch, self.stream, views=False)
        self._step(part, self.batch)
        return self.batch

    def _step(self, part, batch):
        from . import grappa_minibatch_step, minibatch_ws_bytes
        need = minibatch_ws_bytes(batch, self.spec.dims_pad, self.dt)
        if self.mb_ws is None or self.mb_ws.numel() < need:
            self.mb_ws = torch.empty(need + need // 4, dtype=torch.uint8, device=self.dev)
        grappa_minibatch_step(self.ctx, part, batch, self.spec.dims_pad, self.spec.dims[-1],
                              self.theta, self.grad, self.mb_ws, self.loss_dev, self.dt,
                              stream=self.stream, flags=LAYER_NODE_LEVEL if self.corr == "node" else 0)

    def _sample_async(self, part, order, it: int, nb: int):
        from . import Batch, grappa_sample_async
        b = it % nb
        slot = it % len(self.slots)
        seeds = order[b * self.B: min((b + 1) * self.B, order.numel())]
        self.slots[slot] = grappa_sample_async(self.ctx, part, seeds, self.fanouts, self.sample_seed,
                                               self.epoch, b, self.slots[slot] or Batch(),
                                               self.sstreams[it % self.depth])

    def run_epoch(self, on_phase=None):
        """Alg. 1 in mini-batch mode.  Sampling runs `depth` batches ahead on `depth` side streams
        (grappa_sample_async into depth + 1 batch slots), so the samplers of batches i+1 .. i+depth
        run concurrently with each other and with the SAGE step of batch i (the sampler is a chain
        of small latency-bound kernels); the host waits only for batch i's block sizes
        (grappa_sample_wait) before launching its step."""
        from . import grappa_aggregate_grads_c, grappa_epoch_seeds, grappa_sample_wait
        t = self.super_epoch()
        if t != self.t:
            self.repartition(t)
        D = self.depth
        if getattr(self, "sstreams", None) is None:
            self.sstreams = [torch.cuda.Stream(self.dev) for _ in range(D)]
            self.slots = [None] * (D + 1)
        S = len(self.slots)
        for i, w, m_active in phase_plan(self.W, self.G, self.rank):
            part = self.parts.get(w) if w is not None else None
            nb = self.iterations(part)
            iters = self.phase_iterations(part)
            done = [None] * S
            if part is not None:
                if self.order is None or self.order.numel() < part.n_seeds:
                    self.order = torch.empty(part.n_seeds, dtype=torch.int32, device=self.dev)
                order = self.order[:part.n_seeds]
                grappa_epoch_seeds(self.ctx, part, self.sample_seed, self.epoch, order, self.stream)
                ev = torch.cuda.Event()
                ev.record(self.stream)                   # seeds (and every earlier step) first
                for k in range(min(D, iters)):
                    self.sstreams[k % D].wait_event(ev)
                    self._sample_async(part, order, k, nb)
            for it in range(iters):
                slot = it % S
                if part is not None:
                    bt = grappa_sample_wait(self.slots[slot], views=False)
                    nxt = it + D
                    if nxt < iters:
                        if done[nxt % S] is not None:    # that slot's previous blocks are consumed
                            self.sstreams[nxt % D].wait_event(done[nxt % S])
                        self._sample_async(part, order, nxt, nb)
                    self.batch = bt
                    self._step(part, bt)                 # waits on bt's sample event itself
                    done[slot] = torch.cuda.Event()
                    done[slot].record(self.stream)
                    c = bt.factors[self.corr]
                    cov = bt.factors["uniform"]          # the controller's coverage (R32)
                else:
                    self.grad.zero_()
                    c = 0.0
                grappa_aggregate_grads_c(self.ctx, c, self.grad, m_active, self.lr, self.theta,
                                         self.stream, comm_dtype=self.comm_dtype)
                self._steps.append((float(w), cov, 1.0) if part is not None else (0.0, 0.0, 0.0))
                if on_phase is not None:
                    on_phase()
        self.end_epoch()

    def _alloc(self):
        """mini-batch mode needs no partition-sized activation buffers (per-batch workspace
        is sized after each sample)."""
        return None
