"""paper_2602_01872_b200 -- B200-native hot path of Grappa (arXiv 2602.01872).

Thin Python binding over libgrappa.so (C ABI in include/grappa.h).  The functions below
have the ABI's names and only marshal arguments; every step of the path runs in the
sm_100a kernels behind the ABI.  PyTorch provides device memory, streams and process
groups.  ``engine.Trainer`` is the host-side driver (Algorithm 1 phase loop, sweep
schedule, buffers) built on these calls.
"""
from __future__ import annotations

import ctypes
import sys

import torch

from . import _lib
from ._lib import (BF16, BWD_DZ_IN_NORMED, BWD_DZ_OUT_NORMED, CORR, F32, GAT, GCN, LAYER_INPUT, LAYER_NODE_LEVEL, SAGE,
                   GrappaError, load)

__all__ = ["Context", "Part", "Shard", "grappa_shard_extract", "grappa_shard_exchange",
           "grappa_repartition_shards", "grappa_partition", "grappa_repartition", "grappa_layer_fwd",
           "grappa_layer_bwd", "grappa_layer_bwd_ex", "grappa_loss", "grappa_aggregate_grads", "GCN", "SAGE", "F32",
           "BF16", "CORR", "GrappaError", "load"]

_TORCH_DT = {F32: torch.float32, BF16: torch.bfloat16}


def dtype_code(dt) -> int:
    if isinstance(dt, int):          # raw codes pass through (the library validates them)
        return dt
    return {torch.float32: F32, torch.bfloat16: BF16, "f32": F32, "fp32": F32,
            "bf16": BF16}[dt]


def arch_code(a) -> int:
    return {"gcn": GCN, "sage": SAGE, "gat": GAT, GCN: GCN, SAGE: SAGE, GAT: GAT}[a]


class _DevView:
    """Zero-copy __cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str, keepalive):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape),
                                         "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}
        self._keep = keepalive


def _view(ptr, shape, typestr, owner):
    if int(shape[0]) == 0 or not ptr:
        return torch.empty(shape, dtype={"<i4": torch.int32, "<i8": torch.int64,
                                         "<f4": torch.float32}.get(typestr, torch.float32),
                           device="cuda")
    return torch.as_tensor(_DevView(ptr, shape, typestr, owner), device="cuda")


def _torch_alloc(nbytes, stream, user):
    """grappa_alloc_fn over PyTorch's caching allocator (stream-ordered; no cudaFree sync)."""
    try:
        dev = torch.cuda.current_device()
        return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0)) or None
    except Exception:          # out of memory -> NULL -> GRAPPA_E_NOMEM
        return None


def _torch_free(ptr, nbytes, stream, user):
    if ptr and not sys.is_finalizing():
        torch.cuda.caching_allocator_delete(int(ptr))


# module-level: library objects may outlive any one Context and free through these
_ALLOC_CB = _lib.ALLOC_FN(_torch_alloc)
_FREE_CB = _lib.FREE_FN(_torch_free)


class Context:
    """grappa_ctx: one per process + GPU (holds the NCCL communicator when world > 1).  Library-owned
    device memory comes from PyTorch's caching allocator (grappa_ctx_create_ex) unless
    torch_alloc=False (cudaMalloc)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_uid: bytes | None = None,
                 torch_alloc: bool = True):
        lib = load()
        self.lib = lib
        h = ctypes.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = ctypes.create_string_buffer(bytes(nccl_uid), 128)
        if torch_alloc:
            _lib.check("grappa_ctx_create_ex", lib.grappa_ctx_create_ex(device, uid, rank, nranks, _ALLOC_CB,
                                                                        _FREE_CB, None, ctypes.byref(h)))
        else:
            _lib.check("grappa_ctx_create", lib.grappa_ctx_create(device, uid, rank, nranks, ctypes.byref(h)))
        self.h = h
        self.device, self.rank, self.nranks = device, rank, nranks

    def set_variant(self, op: str, variant: int):
        """grappa_set_kernel_variant (tests: cross-check alternative kernels on this ctx)."""
        _lib.check("grappa_set_kernel_variant", self.lib.grappa_set_kernel_variant(self.h, op.encode(), int(variant)))

    def comm_bytes(self):
        """(gradient all-reduce bytes, every other cross-GPU byte) moved by this ctx so far."""
        g, o = ctypes.c_int64(), ctypes.c_int64()
        _lib.check("grappa_comm_bytes", self.lib.grappa_comm_bytes(self.h, ctypes.byref(g), ctypes.byref(o)))
        return g.value, o.value

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _lib.check("grappa_nccl_unique_id", load().grappa_nccl_unique_id(buf))
        return buf.raw

    def launches(self) -> int:
        return int(self.lib.grappa_launch_count(self.h))

    def profile(self, on: bool):
        _lib.check("grappa_profile_enable", self.lib.grappa_profile_enable(self.h, int(on)))

    def profile_read(self, kclass: str):
        """(ms total, calls, algorithmic bytes, flops) of one kernel class since profile(True)."""
        ms, by, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        n = ctypes.c_int64()
        _lib.check("grappa_profile_read", self.lib.grappa_profile_read(
            self.h, _lib.KCLASS[kclass], ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by),
            ctypes.byref(fl)))
        return ms.value, n.value, by.value, fl.value

    def roofline_probe(self, kind: str, nbytes: int, row_bytes: int = 256, iters: int = 5, stream=None) -> float:
        """grappa_roofline_probe: measured GB/s of an HBM copy, an L2-resident read or an
        L2-resident whole-row gather (the SpMM's access pattern without arithmetic)."""
        g = ctypes.c_double()
        _lib.check("grappa_roofline_probe", self.lib.grappa_roofline_probe(
            self.h, _lib.PROBE[kind], int(nbytes), int(row_bytes), int(iters), ctypes.byref(g),
            _lib.stream_ptr(stream)))
        return g.value

    def check(self, stream=None):
        _lib.check("grappa_check", self.lib.grappa_check(self.h, _lib.stream_ptr(stream)))

    def close(self):
        if self.h:
            self.lib.grappa_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        if sys.is_finalizing():      # interpreter exit: the allocator callbacks may be gone; leak
            return
        try:
            self.close()
        except Exception:
            pass


class Part:
    """grappa_part handle + zero-copy tensor views of its device arrays."""

    def __init__(self):
        self.h = ctypes.c_void_p()
        self.info = _lib.PartInfo()

    def refresh(self):
        _lib.check("grappa_part_query", load().grappa_part_query(self.h, ctypes.byref(self.info)))
        I = self.info
        n, m, s = I.n_core, I.nnz, I.n_seeds
        self.n_core, self.nnz, self.n_seeds = n, m, s
        self.rowptr = _view(I.rowptr, (n + 1,), "<i8", self)
        self.col = _view(I.col, (m,), "<i4", self)
        self.core_global = _view(I.core_global, (n,), "<i4", self)
        self.d_l = _view(I.d_l, (n,), "<i4", self)
        self.d_g = _view(I.d_g, (n,), "<i4", self)
        self.norm_gcn = _view(I.norm_gcn, (n,), "<f4", self)
        self.norm_sage = _view(I.norm_sage, (n,), "<f4", self)
        self.seeds = _view(I.seeds, (s,), "<i4", self)
        self.labels = _view(I.labels, (n,), "<i4", self)
        self.node_w = _view(I.node_w, (3, n), "<f4", self)
        self.n_halo = I.n_halo
        self.t_rowptr = _view(I.t_rowptr, (n + 1,), "<i8", self) if I.t_rowptr else None
        self.t_col = _view(I.t_col, (m,), "<i4", self) if I.t_col else None
        if I.feat_dim:
            if I.dtype == BF16:
                self.x = _view(I.x, (n, I.feat_dim), "<i2", self).view(torch.bfloat16)
            else:
                self.x = _view(I.x, (n, I.feat_dim), "<f4", self)
        else:
            self.x = None
        return self

    def host_image(self, reuse: dict | None = None, headroom: float = 0.0):
        """Pinned host buffers for this partition's arrays (grappa_part_host) + the struct.
        reuse: the buffers of an earlier image (e.g. the previous super-epoch's partition of the
        same worker) -- views of them are returned where they are large enough, so a switch
        does not re-pin host memory; new buffers get `headroom` extra capacity."""
        I = self.info
        tdt = torch.bfloat16 if I.dtype == BF16 else torch.float32
        want = dict(rowptr=(I.n_core + 1, torch.int64), col=(I.nnz, torch.int32), d_l=(I.n_core, torch.int32),
                    norm_gcn=(I.n_core, torch.float32), norm_sage=(I.n_core, torch.float32),
                    seeds=(I.n_seeds, torch.int32), labels=(I.n_core, torch.int32),
                    x=(I.n_core * I.feat_dim, tdt), node_w=(3 * I.n_core, torch.float32))
        bufs = {}
        for k, (n, dt) in want.items():
            old = (reuse or {}).get(k)
            base = getattr(old, "_grappa_base", old)
            if base is not None and base.dtype == dt and base.numel() >= n:
                v = base[:n]
            else:
                base = torch.empty(max(n, int(n * (1 + headroom))), dtype=dt, pin_memory=True)
                v = base[:n]
            v._grappa_base = base
            bufs[k] = v
        st = _lib.PartHost(**{k: v.data_ptr() for k, v in bufs.items()})
        return bufs, st

    def download(self, st, stream=None):
        _lib.check("grappa_part_download", load().grappa_part_download(self.h, ctypes.byref(st),
                                                                       _lib.stream_ptr(stream)))

    def upload(self, st, stream=None):
        _lib.check("grappa_part_upload", load().grappa_part_upload(self.h, ctypes.byref(st),
                                                                   _lib.stream_ptr(stream)))

    # ---------------------------------------------------------- images (capacity mode)
    def image_bytes(self) -> int:
        return int(load().grappa_part_image_bytes(self.h))

    def save(self, host: torch.Tensor, stream=None):
        """enqueue D2H of the whole partition into `host` (a pinned uint8 tensor)"""
        _lib.check("grappa_part_save", load().grappa_part_save(
            self.h, ctypes.c_void_p(host.data_ptr()), host.numel(), _lib.stream_ptr(stream)))

    def load_image(self, host: torch.Tensor, stream=None):
        """enqueue H2D of an image into this part's buffers (no host sync)"""
        _lib.check("grappa_part_load", load().grappa_part_load(
            ctypes.byref(self.h), ctypes.c_void_p(host.data_ptr()), _lib.stream_ptr(stream)))
        return self.refresh()

    @staticmethod
    def image_info(host: torch.Tensor):
        info = _lib.PartInfo()
        _lib.check("grappa_part_image_info", load().grappa_part_image_info(
            ctypes.c_void_p(host.data_ptr()), ctypes.byref(info)))
        return info

    def factor(self, corr: str) -> float:
        I = self.info
        return {"none": 1.0, "uniform": I.c_uniform, "resampling": I.c_resampling,
                "resampling_hm": I.c_resampling_hm, "node": 1.0}[corr]

    def destroy(self):
        if self.h:
            load().grappa_part_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        if sys.is_finalizing():      # interpreter exit: the allocator callbacks may be gone; leak
            return
        try:
            self.destroy()
        except Exception:
            pass


def grappa_partition(ctx: Context, num_nodes: int, num_chunks: int, seed: int, chunk_of: torch.Tensor,
                     stream=None):
    sizes = (ctypes.c_int64 * num_chunks)()
    _lib.check("grappa_partition", ctx.lib.grappa_partition(
        ctx.h, num_nodes, num_chunks, ctypes.c_uint64(seed & ((1 << 64) - 1)), _lib.ptr(chunk_of),
        sizes, _lib.stream_ptr(stream)))
    return list(sizes)


def grappa_repartition(ctx: Context, rowptr: torch.Tensor, col: torch.Tensor, feats, dtype,
                       chunk_of: torch.Tensor, num_chunks: int, base: int, swept: int,
                       train_mask: torch.Tensor, labels, part: Part | None = None, stream=None,
                       halo: bool = False) -> Part:
    g = _lib.Csr(rowptr.numel() - 1, col.numel(), rowptr.data_ptr(), col.data_ptr())
    part = part or Part()
    fdim = 0 if feats is None else feats.shape[1]
    _lib.check("grappa_repartition_ex", ctx.lib.grappa_repartition_ex(
        ctx.h, ctypes.byref(g), _lib.ptr(feats), fdim, dtype_code(dtype), _lib.ptr(chunk_of),
        num_chunks, base, swept, _lib.ptr(train_mask), _lib.ptr(labels),
        _lib.PART_HALO1 if halo else 0, ctypes.byref(part.h), _lib.stream_ptr(stream)))
    return part.refresh()


class Index:
    """grappa_index of (global CSR, chunk map): per-edge chunk bytes + per-chunk counts / degree
    sums for grappa_repartition_batch_ix.  Keeps references to the tensors it indexes."""

    def __init__(self, ctx: Context, rowptr: torch.Tensor, col: torch.Tensor, chunk_of: torch.Tensor,
                 num_chunks: int, stream=None):
        self.h = ctypes.c_void_p()
        self.refs = (rowptr, col, chunk_of)
        self.C = num_chunks
        g = _lib.Csr(rowptr.numel() - 1, col.numel(), rowptr.data_ptr(), col.data_ptr())
        _lib.check("grappa_index_create", ctx.lib.grappa_index_create(
            ctx.h, ctypes.byref(g), _lib.ptr(chunk_of), num_chunks, ctypes.byref(self.h), _lib.stream_ptr(stream)))

    def query(self):
        cs, dg = (ctypes.c_int64 * self.C)(), (ctypes.c_int64 * self.C)()
        _lib.check("grappa_index_query", load().grappa_index_query(self.h, cs, dg))
        return list(cs), list(dg)

    def destroy(self):
        if self.h:
            load().grappa_index_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        if sys.is_finalizing():
            return
        try:
            self.destroy()
        except Exception:
            pass


def grappa_repartition_batch(ctx: Context, rowptr: torch.Tensor, col: torch.Tensor, feats, dtype,
                             chunk_of: torch.Tensor, num_chunks: int, pairs, train_mask: torch.Tensor, labels,
                             parts=None, stream=None, chunk_sizes=None, index: "Index" = None) -> list:
    """every partition of a switch (pairs = [(base, swept)] per partition) in one call; parts:
    list of Part (or None) to reuse.  chunk_sizes: grappa_partition's output for chunk_of (computed
    with torch on the device if not given).  index: a prebuilt Index of (rowptr/col, chunk_of)
    (grappa_repartition_batch_ix); None -> the library builds a temporary one."""
    g = _lib.Csr(rowptr.numel() - 1, col.numel(), rowptr.data_ptr(), col.data_ptr())
    K = len(pairs)
    if chunk_sizes is None:
        chunk_sizes = (index.query()[0] if index is not None
                       else torch.bincount(chunk_of.long(), minlength=num_chunks).cpu().tolist())
    cs = (ctypes.c_int64 * num_chunks)(*[int(c) for c in chunk_sizes])
    bs = (ctypes.c_int32 * K)(*[int(b) for b, _ in pairs])
    ss = (ctypes.c_int32 * K)(*[int(s_) for _, s_ in pairs])
    parts = list(parts) if parts is not None else [None] * K
    parts = [p if p is not None else Part() for p in parts]
    hs = (ctypes.c_void_p * K)(*[p.h.value for p in parts])
    fdim = 0 if feats is None else feats.shape[1]
    if index is not None:
        _lib.check("grappa_repartition_batch_ix", ctx.lib.grappa_repartition_batch_ix(
            ctx.h, ctypes.byref(g), _lib.ptr(feats), fdim, dtype_code(dtype), index.h, cs, K, bs, ss,
            _lib.ptr(train_mask), _lib.ptr(labels), hs, _lib.stream_ptr(stream)))
    else:
        _lib.check("grappa_repartition_batch", ctx.lib.grappa_repartition_batch(
            ctx.h, ctypes.byref(g), _lib.ptr(feats), fdim, dtype_code(dtype), _lib.ptr(chunk_of), num_chunks, cs,
            K, bs, ss, _lib.ptr(train_mask), _lib.ptr(labels), hs, _lib.stream_ptr(stream)))
    for p, h in zip(parts, hs):
        p.h = ctypes.c_void_p(h)
        p.refresh()
    return parts


class Shard:
    """grappa_shard handle (one chunk's rows, sharded mode) + views of its device arrays."""

    def __init__(self):
        self.h = ctypes.c_void_p()
        self.info = _lib.ShardInfo()

    def refresh(self):
        _lib.check("grappa_shard_query", load().grappa_shard_query(self.h, ctypes.byref(self.info)))
        I = self.info
        n, m = I.n_rows, I.nnz
        self.chunk, self.n_rows, self.nnz = I.chunk, n, m
        self.ids = _view(I.ids, (n,), "<i4", self)
        self.rowptr = _view(I.rowptr, (n + 1,), "<i8", self)
        self.col = _view(I.col, (m,), "<i4", self)
        self.labels = _view(I.labels, (n,), "<i4", self)
        self.train = _view(I.train, (n,), "|u1", self)
        if I.feat_dim:
            if I.dtype == BF16:
                self.x = _view(I.x, (n, I.feat_dim), "<i2", self).view(torch.bfloat16)
            else:
                self.x = _view(I.x, (n, I.feat_dim), "<f4", self)
        else:
            self.x = None
        return self

    def destroy(self):
        if self.h:
            load().grappa_shard_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        if sys.is_finalizing():      # interpreter exit: the allocator callbacks may be gone; leak
            return
        try:
            self.destroy()
        except Exception:
            pass


def grappa_shard_extract(ctx: Context, rowptr: torch.Tensor, col: torch.Tensor, feats, dtype,
                         chunk_of: torch.Tensor, num_chunks: int, chunk: int, train_mask: torch.Tensor,
                         labels, shard: Shard | None = None, stream=None) -> Shard:
    g = _lib.Csr(rowptr.numel() - 1, col.numel(), rowptr.data_ptr(), col.data_ptr())
    shard = shard or Shard()
    fdim = 0 if feats is None else feats.shape[1]
    _lib.check("grappa_shard_extract", ctx.lib.grappa_shard_extract(
        ctx.h, ctypes.byref(g), _lib.ptr(feats), fdim, dtype_code(dtype), _lib.ptr(chunk_of), num_chunks,
        chunk, _lib.ptr(train_mask), _lib.ptr(labels), ctypes.byref(shard.h), _lib.stream_ptr(stream)))
    return shard.refresh()


def _np_ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def shard_image(rowptr, col, feats, dtype, chunk_of, chunk: int, train_mask, labels, threads: int = 0,
                pin: bool = True) -> torch.Tensor:
    """Host image of chunk `chunk`'s shard (grappa_shard_image_size / _build) from HOST numpy
    arrays (rowptr int64 [N+1], col int32, feats fp32 [N x F_pad] or None, chunk_of int32 [N],
    train_mask uint8, labels int32 or None), in a pinned uint8 tensor."""
    import numpy as np
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    chunk_of = np.ascontiguousarray(chunk_of, dtype=np.int32)
    train_mask = np.ascontiguousarray(train_mask, dtype=np.uint8)
    labels = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    feats = None if feats is None else np.ascontiguousarray(feats, dtype=np.float32)
    N = rowptr.size - 1
    fdim = 0 if feats is None else feats.shape[1]
    n, m, nb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_size_t()
    lib = load()
    _lib.check("grappa_shard_image_size", lib.grappa_shard_image_size(
        _np_ptr(rowptr), N, _np_ptr(chunk_of), chunk, fdim, dtype_code(dtype), ctypes.byref(n), ctypes.byref(m),
        ctypes.byref(nb)))
    img = torch.empty(nb.value, dtype=torch.uint8, pin_memory=pin)
    _lib.check("grappa_shard_image_build", lib.grappa_shard_image_build(
        _np_ptr(rowptr), _np_ptr(col), N, _np_ptr(feats), fdim, dtype_code(dtype), _np_ptr(chunk_of), chunk,
        _np_ptr(train_mask), _np_ptr(labels), ctypes.c_void_p(img.data_ptr()), nb.value, threads))
    return img


def grappa_shard_load(ctx: Context, image: torch.Tensor, shard: Shard | None = None, stream=None) -> Shard:
    """enqueue the H2D copies of a shard image into `shard` (new if None); no host sync"""
    shard = shard or Shard()
    _lib.check("grappa_shard_load", ctx.lib.grappa_shard_load(
        ctx.h, ctypes.c_void_p(image.data_ptr()), ctypes.byref(shard.h), _lib.stream_ptr(stream)))
    return shard.refresh()


def grappa_shard_exchange(ctx: Context, sends, recvs, stream=None):
    """sends: [(peer, Shard)], recvs: [(peer, Shard)] (the receiving Shard objects are filled);
    listed in the order both sides agree on (engine.shard_plan)."""
    n = len(sends) + len(recvs)
    arr = (_lib.ShardXfer * max(n, 1))()
    k = 0
    for peer, sh in sends:
        arr[k] = _lib.ShardXfer(peer, sh.h.value, None)
        k += 1
    for peer, sh in recvs:
        arr[k] = _lib.ShardXfer(peer, None, ctypes.addressof(sh.h))
        k += 1
    _lib.check("grappa_shard_exchange", ctx.lib.grappa_shard_exchange(
        ctx.h, n, ctypes.cast(arr, ctypes.c_void_p), _lib.stream_ptr(stream)))
    for _, sh in recvs:
        sh.refresh()


def grappa_repartition_shards(ctx: Context, base: Shard, swept: Shard, chunk_of: torch.Tensor, num_chunks: int,
                              part: Part | None = None, stream=None, halo: bool = False) -> Part:
    """halo=True: a halo-1 partition whose halo rows are pending until grappa_halo_exchange"""
    part = part or Part()
    _lib.check("grappa_repartition_shards_ex", ctx.lib.grappa_repartition_shards_ex(
        ctx.h, base.h, swept.h, _lib.ptr(chunk_of), chunk_of.numel(), num_chunks, _lib.PART_HALO1 if halo else 0,
        ctypes.byref(part.h), _lib.stream_ptr(stream)))
    return part.refresh()


def grappa_halo_exchange(ctx: Context, part: Part | None, shards, chunk_owner, chunk_of: torch.Tensor,
                         num_chunks: int, stream=None):
    """collective halo feature all-to-all (every rank, once per partition build); shards: the Shard
    objects this rank owns; chunk_owner: rank of each chunk's shard"""
    hs = (ctypes.c_void_p * max(1, len(shards)))(*[sh.h.value for sh in shards])
    own = (ctypes.c_int32 * num_chunks)(*[int(o) for o in chunk_owner])
    _lib.check("grappa_halo_exchange", ctx.lib.grappa_halo_exchange(
        ctx.h, part.h if part is not None else None, len(shards), ctypes.cast(hs, ctypes.c_void_p), own,
        _lib.ptr(chunk_of), num_chunks, _lib.stream_ptr(stream)))
    if part is not None:
        part.refresh()
    return part


def layer_saved_bytes(part: Part, arch, f_in, f_out, dtype, flags: int = 0) -> int:
    return int(load().grappa_layer_saved_bytes_ex(part.h, arch_code(arch), f_in, f_out, dtype_code(dtype),
                                                  int(flags)))


def layer_ws_bytes(part: Part, arch, f_in, f_out, dtype) -> int:
    return int(load().grappa_layer_ws_bytes(part.h, arch_code(arch), f_in, f_out, dtype_code(dtype)))


def grappa_layer_fwd(ctx: Context, part: Part, arch, f_in, f_out, relu, h_in, w, h_out, saved, ws,
                     dtype, stream=None):
    _lib.check("grappa_layer_fwd", ctx.lib.grappa_layer_fwd(
        ctx.h, part.h, arch_code(arch), f_in, f_out, int(relu), _lib.ptr(h_in), _lib.ptr(w),
        _lib.ptr(h_out), _lib.ptr(saved), _lib.ptr(ws), dtype_code(dtype), _lib.stream_ptr(stream)))


def grappa_layer_fwd_ex(ctx: Context, part: Part, arch, f_in, f_out, relu, h_in, w, h_out, saved, ws,
                        dtype, flags: int, stream=None):
    _lib.check("grappa_layer_fwd_ex", ctx.lib.grappa_layer_fwd_ex(
        ctx.h, part.h, arch_code(arch), f_in, f_out, int(relu), _lib.ptr(h_in), _lib.ptr(w),
        _lib.ptr(h_out), _lib.ptr(saved), _lib.ptr(ws), dtype_code(dtype), int(flags),
        _lib.stream_ptr(stream)))


def grappa_layer_bwd(ctx: Context, part: Part, arch, f_in, f_out, relu_in, dz_out, h_in, w, saved,
                     dw, dz_in, ws, dtype, stream=None):
    _lib.check("grappa_layer_bwd", ctx.lib.grappa_layer_bwd(
        ctx.h, part.h, arch_code(arch), f_in, f_out, int(relu_in), _lib.ptr(dz_out), _lib.ptr(h_in),
        _lib.ptr(w), _lib.ptr(saved), _lib.ptr(dw), _lib.ptr(dz_in), _lib.ptr(ws), dtype_code(dtype),
        _lib.stream_ptr(stream)))


def grappa_layer_bwd_ex(ctx: Context, part: Part, arch, f_in, f_out, relu_in, dz_out, h_in, w, saved,
                        dw, dz_in, ws, dtype, flags: int, stream=None):
    _lib.check("grappa_layer_bwd_ex", ctx.lib.grappa_layer_bwd_ex(
        ctx.h, part.h, arch_code(arch), f_in, f_out, int(relu_in), _lib.ptr(dz_out), _lib.ptr(h_in),
        _lib.ptr(w), _lib.ptr(saved), _lib.ptr(dw), _lib.ptr(dz_in), _lib.ptr(ws), dtype_code(dtype),
        int(flags), _lib.stream_ptr(stream)))


def grappa_loss(ctx: Context, part: Part, logits, num_classes, k_pad, dlogits, loss_dev, dtype,
                stream=None, flags: int = 0):
    _lib.check("grappa_loss_ex", ctx.lib.grappa_loss_ex(
        ctx.h, part.h, _lib.ptr(logits), num_classes, k_pad, _lib.ptr(dlogits), _lib.ptr(loss_dev),
        dtype_code(dtype), int(flags), _lib.stream_ptr(stream)))


def grappa_aggregate_grads(ctx: Context, part: Part | None, corr: str, grad, m_active: int, lr: float,
                           theta, stream=None, eps: float = 1e-9, c_max: float = 10.0, comm_dtype="f32"):
    _lib.check("grappa_aggregate_grads", ctx.lib.grappa_aggregate_grads(
        ctx.h, part.h if part is not None else None, CORR[corr], ctypes.c_double(eps), ctypes.c_double(c_max),
        _lib.ptr(grad), grad.numel(), m_active, dtype_code(comm_dtype), ctypes.c_float(lr), _lib.ptr(theta),
        _lib.stream_ptr(stream)))


def grappa_aggregate_grads_c(ctx: Context, c: float, grad, m_active: int, lr: float, theta, stream=None,
                             comm_dtype="f32"):
    _lib.check("grappa_aggregate_grads_c", ctx.lib.grappa_aggregate_grads_c(
        ctx.h, ctypes.c_double(c), _lib.ptr(grad), grad.numel(), m_active, dtype_code(comm_dtype),
        ctypes.c_float(lr), _lib.ptr(theta), _lib.stream_ptr(stream)))


# ------------------------------------------------------------------ a10: mini-batch mode
class Batch:
    """grappa_batch handle (layered blocks of one sampled mini-batch) + tensor views."""

    def __init__(self):
        self.h = ctypes.c_void_p()
        self.blocks = []

    def refresh(self, n_layers: int, views: bool = True):
        lib = load()
        self.blocks = []
        for l in range(n_layers if views else 0):
            bi = _lib.BlockInfo()
            _lib.check("grappa_batch_query", lib.grappa_batch_query(self.h, l, ctypes.byref(bi)))
            self.blocks.append(dict(
                n_dst=bi.n_dst, n_src=bi.n_src, nnz=bi.nnz,
                rowptr=_view(bi.rowptr, (bi.n_dst + 1,), "<i8", self),
                col=_view(bi.col, (bi.nnz,), "<i4", self),
                t_rowptr=_view(bi.t_rowptr, (bi.n_src + 1,), "<i8", self),
                t_col=_view(bi.t_col, (bi.nnz,), "<i4", self),
                inv_cnt=_view(bi.inv_cnt, (bi.n_dst,), "<f4", self),
                inv_cnt_node=_view(bi.inv_cnt_node, (bi.n_dst,), "<f4", self),
                src=_view(bi.src, (bi.n_src,), "<i4", self)))
        cu, cr, ch = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _lib.check("grappa_batch_factors", lib.grappa_batch_factors(
            self.h, ctypes.byref(cu), ctypes.byref(cr), ctypes.byref(ch)))
        self.factors = {"none": 1.0, "uniform": cu.value, "resampling": cr.value,
                        "resampling_hm": ch.value, "node": 1.0}
        return self

    def destroy(self):
        if self.h:
            load().grappa_batch_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        if sys.is_finalizing():      # interpreter exit: the allocator callbacks may be gone; leak
            return
        try:
            self.destroy()
        except Exception:
            pass


def grappa_epoch_seeds(ctx: Context, part: Part, seed: int, epoch: int, order, stream=None):
    _lib.check("grappa_epoch_seeds", ctx.lib.grappa_epoch_seeds(
        ctx.h, part.h, ctypes.c_uint64(seed & ((1 << 64) - 1)), epoch, _lib.ptr(order),
        _lib.stream_ptr(stream)))


def grappa_sample(ctx: Context, part: Part, batch, fanouts, seed: int, epoch: int, batch_index: int,
                  out: Batch | None = None, stream=None, views: bool = True) -> Batch:
    out = out or Batch()
    fan = (ctypes.c_int32 * len(fanouts))(*fanouts)
    _lib.check("grappa_sample", ctx.lib.grappa_sample(
        ctx.h, part.h, _lib.ptr(batch), batch.numel(), fan, len(fanouts),
        ctypes.c_uint64(seed & ((1 << 64) - 1)), epoch, batch_index, ctypes.byref(out.h),
        _lib.stream_ptr(stream)))
    return out.refresh(len(fanouts), views)


def grappa_sample_async(ctx: Context, part: Part, batch, fanouts, seed: int, epoch: int, batch_index: int,
                        out: Batch | None = None, stream=None) -> Batch:
    """enqueue only (no host sync); call grappa_sample_wait(out) before using its blocks"""
    out = out or Batch()
    fan = (ctypes.c_int32 * len(fanouts))(*fanouts)
    _lib.check("grappa_sample_async", ctx.lib.grappa_sample_async(
        ctx.h, part.h, _lib.ptr(batch), batch.numel(), fan, len(fanouts),
        ctypes.c_uint64(seed & ((1 << 64) - 1)), epoch, batch_index, ctypes.byref(out.h),
        _lib.stream_ptr(stream)))
    out.n_layers = len(fanouts)
    return out


def grappa_sample_wait(batch: Batch, views: bool = True) -> Batch:
    _lib.check("grappa_sample_wait", load().grappa_sample_wait(batch.h))
    return batch.refresh(batch.n_layers, views)


def grappa_sample_event(batch: Batch) -> int:
    ev = ctypes.c_void_p()
    _lib.check("grappa_sample_event", load().grappa_sample_event(batch.h, ctypes.byref(ev)))
    return ev.value


def minibatch_ws_bytes(batch: Batch, dims_pad, dtype) -> int:
    dp = (ctypes.c_int32 * len(dims_pad))(*dims_pad)
    return int(load().grappa_minibatch_ws_bytes(batch.h, len(dims_pad) - 1, dp, dtype_code(dtype)))


def grappa_minibatch_step(ctx: Context, part: Part, batch: Batch, dims_pad, num_classes: int, theta,
                          grad, ws, loss_dev, dtype, hidden_out=None, stream=None, flags: int = 0):
    L = len(dims_pad) - 1
    dp = (ctypes.c_int32 * (L + 1))(*dims_pad)
    hid = None
    if hidden_out is not None:
        hid = (ctypes.c_void_p * max(1, L - 1))(*[t.data_ptr() for t in hidden_out])
    _lib.check("grappa_minibatch_step_ex", ctx.lib.grappa_minibatch_step_ex(
        ctx.h, part.h, batch.h, L, dp, num_classes, _lib.ptr(theta), _lib.ptr(grad), _lib.ptr(ws),
        ws.numel() * ws.element_size(), _lib.ptr(loss_dev), hid, dtype_code(dtype), int(flags),
        _lib.stream_ptr(stream)))
