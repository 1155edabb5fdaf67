"""ctypes binding of libgrappa.so -- argument marshalling only, same names as include/grappa.h.

Every function here forwards to the C ABI; no step of the method runs in Python.  Tensors
are torch CUDA tensors passed as raw device pointers.  A missing or unloadable library is a
hard error (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgrappa.so")

F32, BF16 = 0, 1
GCN, SAGE, GAT = 0, 1, 2
CORR = {"none": 0, "uniform": 1, "resampling": 2, "resampling_hm": 3, "node": 4}
BWD_DZ_OUT_NORMED, BWD_DZ_IN_NORMED = 1, 2
LAYER_NODE_LEVEL = 4
LAYER_INPUT = 8
PART_HALO1 = 1
PROBE = {"hbm_copy": 0, "l2_read": 1, "l2_gather": 2}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_SHAPE", 3: "E_EMPTY", 4: "E_NONFINITE", 5: "E_SUPPORT",
          6: "E_NOMEM", 7: "E_CUDA", 8: "E_NCCL"}

# every symbol include/grappa.h declares
SYMBOLS = ["grappa_version", "grappa_last_error", "grappa_nccl_unique_id", "grappa_ctx_create",
           "grappa_ctx_destroy", "grappa_partition", "grappa_repartition", "grappa_part_query",
           "grappa_part_destroy", "grappa_layer_saved_bytes", "grappa_layer_ws_bytes",
           "grappa_layer_fwd", "grappa_layer_bwd", "grappa_loss", "grappa_aggregate_grads",
           "grappa_check", "grappa_launch_count", "grappa_profile_enable", "grappa_profile_read",
           "grappa_set_kernel_variant", "grappa_aggregate_grads_c", "grappa_epoch_seeds",
           "grappa_sample", "grappa_batch_query", "grappa_batch_factors", "grappa_batch_destroy",
           "grappa_minibatch_ws_bytes", "grappa_minibatch_step", "grappa_part_download",
           "grappa_part_upload", "grappa_layer_bwd_ex", "grappa_layer_fwd_ex",
           "grappa_minibatch_step_ex", "grappa_sample_async", "grappa_sample_wait",
           "grappa_sample_event", "grappa_repartition_ex", "grappa_part_image_bytes",
           "grappa_part_save", "grappa_part_image_info", "grappa_part_load", "grappa_layer_saved_bytes_ex",
           "grappa_loss_ex", "grappa_shard_extract", "grappa_shard_query", "grappa_shard_destroy",
           "grappa_shard_exchange", "grappa_repartition_shards", "grappa_roofline_probe",
           "grappa_ctx_create_ex", "grappa_comm_bytes", "grappa_repartition_batch",
           "grappa_index_create", "grappa_index_query", "grappa_index_destroy", "grappa_repartition_batch_ix",
           "grappa_shard_image_size", "grappa_shard_image_build", "grappa_shard_load",
           "grappa_repartition_shards_ex", "grappa_halo_exchange"]
KCLASS = {"spmm": 0, "gemm": 1, "gemm_tn": 2, "loss": 3, "agg": 4, "repart": 5, "sample": 6}


# caller allocator callbacks (grappa_ctx_create_ex): void* alloc(size_t, void* stream, void* user),
# void free(void* ptr, size_t, void* stream, void* user)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


class GrappaError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


class Csr(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p)]


class PartInfo(ctypes.Structure):
    _fields_ = [("n_core", ctypes.c_int64), ("nnz", ctypes.c_int64), ("n_seeds", ctypes.c_int64),
                ("base", ctypes.c_int32), ("swept", ctypes.c_int32), ("feat_dim", ctypes.c_int32),
                ("dtype", ctypes.c_int),
                ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("core_global", ctypes.c_void_p), ("d_l", ctypes.c_void_p), ("d_g", ctypes.c_void_p),
                ("norm_gcn", ctypes.c_void_p), ("norm_sage", ctypes.c_void_p),
                ("seeds", ctypes.c_void_p), ("labels", ctypes.c_void_p), ("x", ctypes.c_void_p),
                ("n_heavy", ctypes.c_int64), ("n_slots", ctypes.c_int64),
                ("c_uniform", ctypes.c_double), ("c_resampling", ctypes.c_double),
                ("c_resampling_hm", ctypes.c_double), ("D", ctypes.c_int64),
                ("node_w", ctypes.c_void_p), ("n_halo", ctypes.c_int64),
                ("t_rowptr", ctypes.c_void_p), ("t_col", ctypes.c_void_p)]


class ShardInfo(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_int32), ("feat_dim", ctypes.c_int32), ("dtype", ctypes.c_int),
                ("n_rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("ids", ctypes.c_void_p), ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("x", ctypes.c_void_p), ("labels", ctypes.c_void_p), ("train", ctypes.c_void_p)]


class ShardXfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("send", ctypes.c_void_p), ("recv", ctypes.c_void_p)]


class PartHost(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("rowptr", "col", "d_l", "norm_gcn", "norm_sage", "seeds", "labels", "x", "node_w")]


class BlockInfo(ctypes.Structure):
    _fields_ = [("n_dst", ctypes.c_int32), ("n_src", ctypes.c_int32), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("t_rowptr", ctypes.c_void_p), ("t_col", ctypes.c_void_p),
                ("inv_cnt", ctypes.c_void_p), ("src", ctypes.c_void_p),
                ("inv_cnt_node", ctypes.c_void_p)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libgrappa.so (never builds implicitly; __graft_entry__.build() does that)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    vp, i32, i64, u64, f32, dbl, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_float, ctypes.c_double,
                                        ctypes.c_size_t)
    st = ctypes.c_int
    sig = {
        "grappa_version": (ctypes.c_char_p, []),
        "grappa_last_error": (ctypes.c_char_p, []),
        "grappa_nccl_unique_id": (st, [vp]),
        "grappa_ctx_create": (st, [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]),
        "grappa_ctx_destroy": (None, [vp]),
        "grappa_partition": (st, [vp, i64, i32, u64, vp, vp, vp]),
        "grappa_repartition": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.c_int, vp, i32, i32,
                                    i32, vp, vp, ctypes.POINTER(vp), vp]),
        "grappa_repartition_ex": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.c_int, vp, i32, i32,
                                       i32, vp, vp, ctypes.c_uint, ctypes.POINTER(vp), vp]),
        "grappa_part_query": (st, [vp, ctypes.POINTER(PartInfo)]),
        "grappa_shard_extract": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.c_int, vp, i32, i32, vp, vp,
                                      ctypes.POINTER(vp), vp]),
        "grappa_shard_query": (st, [vp, ctypes.POINTER(ShardInfo)]),
        "grappa_shard_destroy": (None, [vp]),
        "grappa_shard_exchange": (st, [vp, i32, vp, vp]),
        "grappa_repartition_shards": (st, [vp, vp, vp, vp, i64, i32, ctypes.POINTER(vp), vp]),
        "grappa_part_image_bytes": (sz, [vp]),
        "grappa_part_save": (st, [vp, vp, sz, vp]),
        "grappa_part_image_info": (st, [vp, ctypes.POINTER(PartInfo)]),
        "grappa_part_load": (st, [ctypes.POINTER(vp), vp, vp]),
        "grappa_part_destroy": (None, [vp]),
        "grappa_layer_saved_bytes": (sz, [vp, ctypes.c_int, i32, i32, ctypes.c_int]),
        "grappa_layer_ws_bytes": (sz, [vp, ctypes.c_int, i32, i32, ctypes.c_int]),
        "grappa_layer_saved_bytes_ex": (sz, [vp, ctypes.c_int, i32, i32, ctypes.c_int, ctypes.c_uint]),
        "grappa_layer_fwd": (st, [vp, vp, ctypes.c_int, i32, i32, ctypes.c_int, vp, vp, vp, vp, vp,
                                  ctypes.c_int, vp]),
        "grappa_layer_bwd": (st, [vp, vp, ctypes.c_int, i32, i32, ctypes.c_int, vp, vp, vp, vp, vp,
                                  vp, vp, ctypes.c_int, vp]),
        "grappa_layer_bwd_ex": (st, [vp, vp, ctypes.c_int, i32, i32, ctypes.c_int, vp, vp, vp, vp, vp,
                                     vp, vp, ctypes.c_int, ctypes.c_uint, vp]),
        "grappa_layer_fwd_ex": (st, [vp, vp, ctypes.c_int, i32, i32, ctypes.c_int, vp, vp, vp, vp, vp,
                                     ctypes.c_int, ctypes.c_uint, vp]),
        "grappa_loss": (st, [vp, vp, vp, i32, i32, vp, vp, ctypes.c_int, vp]),
        "grappa_loss_ex": (st, [vp, vp, vp, i32, i32, vp, vp, ctypes.c_int, ctypes.c_uint, vp]),
        "grappa_aggregate_grads": (st, [vp, vp, ctypes.c_int, dbl, dbl, vp, i64, i32, ctypes.c_int, f32, vp, vp]),
        "grappa_repartition_batch": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.c_int, vp, i32, vp, i32, vp, vp,
                                          vp, vp, vp, vp]),
        "grappa_repartition_batch_ix": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.c_int, vp, vp, i32, vp, vp,
                                             vp, vp, vp, vp]),
        "grappa_index_create": (st, [vp, ctypes.POINTER(Csr), vp, i32, ctypes.POINTER(vp), vp]),
        "grappa_shard_image_size": (st, [vp, i64, vp, i32, i32, ctypes.c_int, ctypes.POINTER(i64),
                                         ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_size_t)]),
        "grappa_shard_image_build": (st, [vp, vp, i64, vp, i32, ctypes.c_int, vp, i32, vp, vp, vp, ctypes.c_size_t,
                                          i32]),
        "grappa_shard_load": (st, [vp, vp, ctypes.POINTER(vp), vp]),
        "grappa_repartition_shards_ex": (st, [vp, vp, vp, vp, i64, i32, ctypes.c_uint, ctypes.POINTER(vp), vp]),
        "grappa_halo_exchange": (st, [vp, vp, i32, vp, vp, vp, i32, vp]),
        "grappa_index_query": (st, [vp, vp, vp]),
        "grappa_index_destroy": (None, [vp]),
        "grappa_comm_bytes": (st, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "grappa_ctx_create_ex": (st, [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ALLOC_FN, FREE_FN, vp,
                                      ctypes.POINTER(vp)]),
        "grappa_check": (st, [vp, vp]),
        "grappa_launch_count": (i64, [vp]),
        "grappa_profile_enable": (st, [vp, ctypes.c_int]),
        "grappa_set_kernel_variant": (st, [vp, ctypes.c_char_p, ctypes.c_int]),
        "grappa_part_download": (st, [vp, ctypes.POINTER(PartHost), vp]),
        "grappa_part_upload": (st, [vp, ctypes.POINTER(PartHost), vp]),
        "grappa_aggregate_grads_c": (st, [vp, dbl, vp, i64, i32, ctypes.c_int, f32, vp, vp]),
        "grappa_epoch_seeds": (st, [vp, vp, u64, i64, vp, vp]),
        "grappa_sample": (st, [vp, vp, vp, i32, vp, i32, u64, i64, i64, ctypes.POINTER(vp), vp]),
        "grappa_sample_async": (st, [vp, vp, vp, i32, vp, i32, u64, i64, i64, ctypes.POINTER(vp), vp]),
        "grappa_sample_wait": (st, [vp]),
        "grappa_sample_event": (st, [vp, ctypes.POINTER(vp)]),
        "grappa_batch_query": (st, [vp, i32, ctypes.POINTER(BlockInfo)]),
        "grappa_batch_factors": (st, [vp, ctypes.POINTER(dbl), ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "grappa_batch_destroy": (None, [vp]),
        "grappa_minibatch_ws_bytes": (sz, [vp, i32, vp, ctypes.c_int]),
        "grappa_minibatch_step": (st, [vp, vp, vp, i32, vp, i32, vp, vp, vp, sz, vp, vp, ctypes.c_int, vp]),
        "grappa_minibatch_step_ex": (st, [vp, vp, vp, i32, vp, i32, vp, vp, vp, sz, vp, vp, ctypes.c_int,
                                          ctypes.c_uint, vp]),
        "grappa_roofline_probe": (st, [vp, ctypes.c_int, i64, i32, i32, ctypes.POINTER(dbl), vp]),
        "grappa_profile_read": (st, [vp, ctypes.c_int, ctypes.POINTER(dbl), ctypes.POINTER(i64),
                                     ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(fn: str, status: int):
    if status != 0:
        msg = load().grappa_last_error().decode(errors="replace")
        raise GrappaError(fn, status, msg)


def ptr(t) -> ctypes.c_void_p:
    """Raw data pointer of a torch tensor (or None)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream if stream is not None else 0)
