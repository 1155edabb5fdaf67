"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench, tests).

This module holds none of the method's arithmetic: it only turns a root seed into
graphs (CSR), features, labels, train masks and initial weights, per the recipe in
DESIGN.md §3.  The heavy lifting is in ``gen.c`` (C + OpenMP, thread-count independent);
this file is ctypes marshalling plus the workload table (BASELINE.json ``configs``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_gen.so")
_lib = None

ROOT_SEED = 0x6772617070610001
TAGS = {"graph": 1, "perm": 2, "chunks": 3, "feat": 4, "label": 5, "split": 6,
        "init": 7, "sample": 8, "dropout": 9}
M64 = (1 << 64) - 1


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_SO)
    u64, i64, i32, dbl, vp = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32,
                              ctypes.c_double, ctypes.c_void_p)
    lib.gen_mix.restype = u64; lib.gen_mix.argtypes = [u64]
    lib.gen_h2.restype = u64; lib.gen_h2.argtypes = [u64, u64]
    lib.gen_h3.restype = u64; lib.gen_h3.argtypes = [u64, u64, u64]
    lib.gen_rmat.restype = i64
    lib.gen_rmat.argtypes = [ctypes.c_int, i64, i64, dbl, dbl, dbl, u64, u64, vp,
                             ctypes.POINTER(vp)]
    lib.gen_sbm.restype = i64
    lib.gen_sbm.argtypes = [i64, vp, dbl, dbl, u64, vp, ctypes.POINTER(vp)]
    lib.gen_free.argtypes = [vp]
    lib.gen_features.argtypes = [i64, i32, i32, u64, vp, ctypes.c_float, vp]
    lib.gen_labels.argtypes = [i64, i32, u64, vp]
    lib.gen_train_mask.argtypes = [i64, u64, u64, vp]
    lib.gen_glorot.argtypes = [i32, i32, i32, i32, u64, u64, u64, vp]
    lib.gen_scramble.argtypes = [i64, u64, vp, vp, i64]
    lib.gen_num_threads.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- hashing (scalar)
def mix(x: int) -> int:
    return int(_load().gen_mix(x & M64))


def h(*args: int) -> int:
    """h(a, b, c, ...) = mix(a ^ mix(b ^ mix(c ^ ...))), innermost argument first."""
    acc = mix(args[-1] & M64)
    for a in reversed(args[:-1]):
        acc = mix((a & M64) ^ acc)
    return acc


def seed_of(tag: str, root: int = ROOT_SEED) -> int:
    return h(root, TAGS[tag])


def scramble(n: int, seed: int, ids: np.ndarray) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty_like(ids)
    _load().gen_scramble(n, seed, _ptr(ids), _ptr(out), ids.size)
    return out


def pad16(d: int) -> int:
    return (d + 15) // 16 * 16


# ---------------------------------------------------------------- graphs
def _take_csr(n: int, nnz: int, rowptr: np.ndarray, colp: ctypes.c_void_p) -> tuple:
    lib = _load()
    col = np.empty(nnz, dtype=np.int32)
    if nnz:
        ctypes.memmove(col.ctypes.data, colp.value, nnz * 4)
    lib.gen_free(colp)
    return rowptr, col


def rmat(scale: int, n: int, num_samples: int, seed_graph: int, seed_perm: int,
         abc=(0.57, 0.19, 0.19)) -> tuple:
    """Undirected RMAT CSR (rowptr int64[n+1], col int32[nnz]); see gen.c."""
    lib = _load()
    rowptr = np.empty(n + 1, dtype=np.int64)
    colp = ctypes.c_void_p()
    nnz = lib.gen_rmat(scale, n, num_samples, abc[0], abc[1], abc[2], seed_graph, seed_perm,
                       _ptr(rowptr), ctypes.byref(colp))
    return _take_csr(n, nnz, rowptr, colp)


def sbm(community: np.ndarray, p_in: float, p_out: float, seed_graph: int) -> tuple:
    lib = _load()
    community = np.ascontiguousarray(community, dtype=np.int32)
    n = community.size
    rowptr = np.empty(n + 1, dtype=np.int64)
    colp = ctypes.c_void_p()
    nnz = lib.gen_sbm(n, _ptr(community), p_in, p_out, seed_graph, _ptr(rowptr),
                      ctypes.byref(colp))
    return _take_csr(n, nnz, rowptr, colp)


def csr_from_edges(n: int, edges) -> tuple:
    """Tiny helper for hand-built test graphs: undirected edge list -> canonical CSR."""
    adj = [set() for _ in range(n)]
    for u, v in edges:
        if u != v:
            adj[u].add(v); adj[v].add(u)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for v in range(n):
        nb = sorted(adj[v])
        cols.extend(nb)
        rowptr[v + 1] = rowptr[v] + len(nb)
    return rowptr, np.asarray(cols, dtype=np.int32)


# ---------------------------------------------------------------- node data
def features(n: int, F: int, F_pad: int, seed: int, community=None, signal: float = 0.0):
    x = np.empty((n, F_pad), dtype=np.float32)
    comm = None if community is None else np.ascontiguousarray(community, dtype=np.int32)
    _load().gen_features(n, F, F_pad, seed, None if comm is None else _ptr(comm),
                         float(signal), _ptr(x))
    return x


def labels(n: int, K: int, seed: int) -> np.ndarray:
    y = np.empty(n, dtype=np.int32)
    _load().gen_labels(n, K, seed, _ptr(y))
    return y


def train_mask(n: int, frac: float, seed: int) -> np.ndarray:
    m = np.empty(n, dtype=np.uint8)
    thr = M64 if frac >= 1.0 else int(frac * 2.0 ** 64)
    _load().gen_train_mask(n, seed, thr, _ptr(m))
    return m


def glorot(fan_in: int, fan_out: int, rows_pad: int, cols_pad: int, seed: int, layer: int,
           mat: int) -> np.ndarray:
    w = np.empty((rows_pad, cols_pad), dtype=np.float32)
    _load().gen_glorot(fan_in, fan_out, rows_pad, cols_pad, seed, layer, mat, _ptr(w))
    return w


def num_threads() -> int:
    return int(_load().gen_num_threads())


# ---------------------------------------------------------------- workloads
@dataclass
class Workload:
    """One synthetic dataset + model shape (BASELINE.json ``configs``)."""
    name: str
    kind: str                    # "rmat" | "sbm"
    n: int
    F: int
    K: int
    arch: str                    # "gcn" | "sage" | "gat"
    depth: int
    hidden: int = 128
    train_frac: float = 0.1
    scale: int = 0
    num_samples: int = 0
    chunks: int = 8
    correction: str = "resampling"
    repartition_every: int = 10
    sbm_sizes: tuple = ()
    p_in: float = 0.0
    p_out: float = 0.0
    root: int = ROOT_SEED
    extra: dict = field(default_factory=dict)

    @property
    def dims(self):
        return [self.F] + [self.hidden] * (self.depth - 1) + [self.K]

    @property
    def dims_pad(self):
        return [pad16(d) for d in self.dims]


WORKLOADS = {
    # configs[0]: Cora-shaped SBM, GCN-2, 2 partitions (C=2 degenerate, C=4 real isolation)
    "cora": Workload("cora", "sbm", 2708, 1433, 7, "gcn", 2, train_frac=0.0, chunks=2,
                     sbm_sizes=(387,) * 6 + (386,), p_in=8.08e-3, p_out=3.36e-4),
    # configs[1]: ogbn-arxiv-shaped RMAT, SAGE-3, 8 partitions, shrinkage
    "arxiv": Workload("arxiv", "rmat", 169_343, 128, 40, "sage", 3, train_frac=0.537,
                      scale=18, num_samples=1_237_000, chunks=8),
    # configs[2]: ogbn-products-shaped RMAT, GCN-8, 8 partitions, repartition every N epochs
    "products": Workload("products", "rmat", 2_449_029, 100, 47, "gcn", 8, train_frac=0.0803,
                         scale=22, num_samples=65_800_000, chunks=8, repartition_every=10),
    # configs[3]: ogbn-papers100M-shaped RMAT, SAGE-3 mini-batch (B = 1000, fanouts
    # {15,10,5} input -> output, R25), 8 partitions
    "papers": Workload("papers", "rmat", 111_059_956, 128, 172, "sage", 3, train_frac=0.01087,
                       scale=27, num_samples=1_666_000_000, chunks=8,
                       extra=dict(mode="minibatch", fanouts=(15, 10, 5), batch_size=1000)),
    # configs[4]: R-MAT scaling sweep (Graph500, edge factor 16), GCN-4, min-distance
    # (uniform) correction, W = C partitions
    "rmat22": Workload("rmat22", "rmat", 1 << 22, 128, 16, "gcn", 4, train_frac=0.1, scale=22,
                       num_samples=1 << 26, chunks=8, correction="uniform"),
    "rmat24": Workload("rmat24", "rmat", 1 << 24, 128, 16, "gcn", 4, train_frac=0.1, scale=24,
                       num_samples=1 << 28, chunks=8, correction="uniform"),
    "rmat26": Workload("rmat26", "rmat", 1 << 26, 128, 16, "gcn", 4, train_frac=0.1, scale=26,
                       num_samples=1 << 30, chunks=8, correction="uniform"),
}
# §8f row 4: the products graph under GAT-3 (R35), full-graph, P = 8 (not a BASELINE config)
WORKLOADS["products_gat"] = Workload(**{**WORKLOADS["products"].__dict__, "name": "products_gat",
                                        "arch": "gat", "depth": 3})
WORKLOADS["cora4"] = Workload(**{**WORKLOADS["cora"].__dict__, "name": "cora4", "chunks": 4,
                                 "extra": dict(workers=2)})


def small_workload(name: str, n: int, scale: int, num_samples: int, **kw) -> Workload:
    """Scaled-down instance of a workload's generator (parity-test sizes)."""
    base = WORKLOADS[name]
    d = dict(base.__dict__)
    d.update(dict(name=f"{name}-small", n=n, scale=scale, num_samples=num_samples))
    d.update(kw)
    return Workload(**d)


@dataclass
class Dataset:
    wl: Workload
    rowptr: np.ndarray
    col: np.ndarray
    x: np.ndarray            # [n, F_pad] float32, padded columns zero
    y: np.ndarray            # [n] int32
    train: np.ndarray        # [n] uint8
    weights: list            # per layer: list of fp32 [fin_pad, fout_pad] (GCN: [W]; SAGE: [W_self, W_nbr])

    @property
    def nnz(self):
        return int(self.rowptr[-1])


def make_dataset(wl: Workload, with_features: bool = True) -> Dataset:
    root = wl.root
    sg, sp, sf, sl, ss, si = (seed_of(t, root) for t in
                              ("graph", "perm", "feat", "label", "split", "init"))
    if wl.kind == "sbm":
        comm = np.concatenate([np.full(s, c, dtype=np.int32) for c, s in enumerate(wl.sbm_sizes)])
        assert comm.size == wl.n
        rowptr, col = sbm(comm, wl.p_in, wl.p_out, sg)
        y = comm.copy()
        # train: the 20 lowest-hash nodes of every community
        hv = np.array([h(ss, v) for v in range(wl.n)], dtype=np.uint64)
        train = np.zeros(wl.n, dtype=np.uint8)
        for c in range(len(wl.sbm_sizes)):
            idx = np.nonzero(comm == c)[0]
            order = idx[np.lexsort((idx, hv[idx]))]
            train[order[:20]] = 1
        x = features(wl.n, wl.F, pad16(wl.F), sf, comm, 1.0) if with_features else None
    else:
        rowptr, col = rmat(wl.scale, wl.n, wl.num_samples, sg, sp)
        y = labels(wl.n, wl.K, sl)
        train = train_mask(wl.n, wl.train_frac, ss)
        x = features(wl.n, wl.F, pad16(wl.F), sf) if with_features else None
    weights = init_weights(wl, si)
    return Dataset(wl, rowptr, col, x, y, train, weights)


def shared_dataset(wl: Workload, rank: int, barrier, root: str = "/dev/shm") -> Dataset:
    """One copy of a dataset for all ranks of a node: rank 0 generates it and writes the arrays to
    `root` (page cache, shared), the others wait at `barrier()` and map them read-only.  Avoids N
    concurrent generations and N private host copies (8 x 57 GB of fp32 features at papers
    scale).  Falls back to a private generation when `root` is not writable."""
    import hashlib
    key = hashlib.sha1(repr(sorted(wl.__dict__.items())).encode()).hexdigest()[:12]
    base = os.path.join(root, f"grappa_{wl.name}_{key}")
    names = ("rowptr", "col", "x", "y", "train")
    ok = os.path.isdir(root) and os.access(root, os.W_OK)
    if rank == 0:
        ds = make_dataset(wl)
        if ok:
            try:
                for n in names:
                    np.save(f"{base}_{n}.tmp.npy", getattr(ds, n))
                    os.replace(f"{base}_{n}.tmp.npy", f"{base}_{n}.npy")
            except OSError:
                ok = False
        barrier()
        return ds
    barrier()
    if ok and all(os.path.exists(f"{base}_{n}.npy") for n in names):
        arr = {n: np.load(f"{base}_{n}.npy", mmap_mode="r") for n in names}
        return Dataset(wl, arr["rowptr"], arr["col"], arr["x"], arr["y"], arr["train"],
                       init_weights(wl, seed_of("init", wl.root)))
    return make_dataset(wl)


def init_weights(wl: Workload, seed: int) -> list:
    dims, dp = wl.dims, wl.dims_pad
    out = []
    for l in range(wl.depth):
        if wl.arch == "gat":     # [W, [a_src; a_dst]] (2 x f_out attention vectors, glorot)
            out.append([glorot(dims[l], dims[l + 1], dp[l], dp[l + 1], seed, l, 0),
                        glorot(2, dims[l + 1], 2, dp[l + 1], seed, l, 1)])
            continue
        mats = 1 if wl.arch == "gcn" else 2
        out.append([glorot(dims[l], dims[l + 1], dp[l], dp[l + 1], seed, l, m)
                    for m in range(mats)])
    return out
