"""Sharded mode of a3 (P:198 chunks, "workers load the new
chunk's edges"): chunk shards cut out bit-exactly, shipped through NCCL point-to-point
(a 1-rank communicator's self transfer on this single-GPU box), and the partition built from two
shards equal -- bit for bit -- to the oracle's induced partition; a sharded training run equals
the replicated one bit for bit."""
import math

import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import partition as Po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


@pytest.fixture(scope="module")
def prod():
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3)
    return gen.make_dataset(wl)


def upload(ds, dtype=torch.float32):
    d = "cuda"
    return (torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d),
            torch.from_numpy(ds.x).to(d).to(dtype), torch.from_numpy(ds.y).to(d),
            torch.from_numpy(ds.train).to(d))


def shards_of(G, ctx, ds, C, dtype="f32"):
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rp, col, x, y, tr = upload(ds, tdt)
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device="cuda")
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    return ch, {c: G.grappa_shard_extract(ctx, rp, col, x, dtype, ch, C, c, tr, y) for c in range(C)}


@pytest.mark.parametrize("C", [2, 8])
def test_shard_extract_bitexact(G, prod, C):
    ctx = G.Context(0)
    ds = prod
    ch, sh = shards_of(G, ctx, ds, C)
    chunk_of = Po.make_chunks(ds.wl.n, C, gen.seed_of("chunks"))
    for c, s in sh.items():
        ids = np.flatnonzero(chunk_of == c)
        deg = ds.rowptr[ids + 1] - ds.rowptr[ids]
        assert s.chunk == c and np.array_equal(s.ids.cpu().numpy(), ids)
        assert np.array_equal(s.rowptr.cpu().numpy(), np.concatenate([[0], np.cumsum(deg)]))
        ref_col = np.concatenate([ds.col[ds.rowptr[v]:ds.rowptr[v + 1]] for v in ids])
        assert np.array_equal(s.col.cpu().numpy(), ref_col)
        assert np.array_equal(s.labels.cpu().numpy(), ds.y[ids])
        assert np.array_equal(s.train.cpu().numpy(), ds.train[ids].astype(np.uint8))
        assert np.array_equal(s.x.cpu().numpy(), ds.x[ids])
    assert sum(s.n_rows for s in sh.values()) == ds.wl.n
    assert sum(s.nnz for s in sh.values()) == ds.col.size
    with pytest.raises(G.GrappaError, match="E_ARG"):
        rp, col, x, y, tr = upload(ds)
        G.grappa_shard_extract(ctx, rp, col, x, "f32", ch, C, C, tr, y)
    ctx.close()


@pytest.mark.parametrize("C,pairs,dtype", [(8, [(0, 1), (3, 7), (6, 2)], "f32"), (2, [(0, 1)], "bf16"),
                                            (4, [(1, 3), (3, 1)], "f32")])
def test_repartition_shards_bitexact(G, prod, C, pairs, dtype):
    """partition from two shards == the oracle's induced partition (every array, the coverage
    statistics) == the replicated path's partition (SpMM plan included)"""
    ctx = G.Context(0)
    ds = prod
    ch, sh = shards_of(G, ctx, ds, C, dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rp, col, x, y, tr = upload(ds, tdt)
    chunk_of = Po.make_chunks(ds.wl.n, C, gen.seed_of("chunks"))
    part = None
    for b, s in pairs:
        part = G.grappa_repartition_shards(ctx, sh[b], sh[s], ch, C, part)
        rep = G.grappa_repartition(ctx, rp, col, x, dtype, ch, C, b, s, tr, y)
        ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
        assert (part.info.base, part.info.swept) == (b, s)
        assert np.array_equal(part.core_global.cpu().numpy(), ref["core"])
        assert np.array_equal(part.rowptr.cpu().numpy(), ref["rowptr"])
        assert np.array_equal(part.col.cpu().numpy(), ref["col"])
        assert np.array_equal(part.d_l.cpu().numpy(), ref["d_l"])
        assert np.array_equal(part.d_g.cpu().numpy(), ref["d_g"])
        assert np.array_equal(part.seeds.cpu().numpy(), ref["seeds"])
        assert np.array_equal(part.labels.cpu().numpy(), ds.y[ref["core"]])
        xr = torch.from_numpy(ds.x[ref["core"]]).to(tdt)
        assert torch.equal(part.x.cpu().view(torch.int16 if dtype == "bf16" else torch.int32),
                           xr.view(torch.int16 if dtype == "bf16" else torch.int32))
        s_dl, s_dg = ref["d_l"][ref["seeds"]], ref["d_g"][ref["seeds"]]
        assert part.info.D == int(np.sum((s_dg - s_dl)[s_dl > 0]))
        assert part.info.c_resampling == Co.c_resampling(s_dl, s_dg)
        assert math.isclose(part.info.c_uniform, Co.c_uniform(s_dl, s_dg), rel_tol=1e-12)
        for k in ("norm_gcn", "norm_sage", "node_w"):
            assert torch.equal(getattr(part, k), getattr(rep, k)), k
        assert (part.info.n_heavy, part.info.n_slots) == (rep.info.n_heavy, rep.info.n_slots)
        assert part.info.c_uniform == rep.info.c_uniform
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_repartition_shards(ctx, sh[pairs[0][0]], sh[pairs[0][0]], ch, C)
    ctx.close()


def test_shard_exchange_self_nccl(G, prod):
    """grappa_shard_exchange through NCCL (a 1-rank communicator: send to and receive from
    itself in one group) delivers the shard byte for byte, into a fresh and a reused slot"""
    uid = G.Context.nccl_unique_id()
    ctx = G.Context(0, rank=0, nranks=1, nccl_uid=uid)
    ds = prod
    ch, sh = shards_of(G, ctx, ds, 4, "bf16")
    slot = G.Shard()
    for c in (2, 0):                          # second round reuses (grows) the slot
        G.grappa_shard_exchange(ctx, [(0, sh[c])], [(0, slot)])
        torch.cuda.synchronize()
        assert slot.chunk == c and slot.n_rows == sh[c].n_rows and slot.nnz == sh[c].nnz
        for k in ("ids", "rowptr", "col", "labels", "train"):
            assert torch.equal(getattr(slot, k), getattr(sh[c], k)), k
        assert torch.equal(slot.x.view(torch.int16), sh[c].x.view(torch.int16))
    # the received shard feeds the repartition like a local one
    p1 = G.grappa_repartition_shards(ctx, sh[1], slot, ch, 4)
    p2 = G.grappa_repartition_shards(ctx, sh[1], sh[0], ch, 4)
    assert torch.equal(p1.col, p2.col) and torch.equal(p1.core_global, p2.core_global)
    ctx.check()
    ctx.close()
    # no communicator -> E_ARG, not a hang
    c0 = G.Context(0)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_shard_exchange(c0, [(0, sh[1])], [(0, G.Shard())])
    c0.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_sharded_training_equals_replicated(G, prod, dtype):
    """Alg. 1 epochs over two super-epoch switches: the sharded trainer (owned shards only, the
    replicated graph dropped) reproduces the replicated trainer's theta bit for bit"""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda sharded: Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                                 gen.seed_of("chunks"), corr="resampling_hm", lr=0.05, repartition_every=1,
                                 dtype=dtype, sharded=sharded)
    a, b = mk(False), mk(True)
    assert b.rowptr is None and len(b.shards) == wl.chunks      # G = 1: this rank owns every chunk
    for _ in range(2):
        a.run_epoch()
        b.run_epoch()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(a.theta, b.theta)
    assert a.losses == b.losses
    ctx.close()


@pytest.mark.parametrize("dtype,nccl", [("f32", True), ("bf16", True), ("bf16", False)])
def test_sharded_halo_partition_bitexact(G, prod, dtype, nccl):
    """§8f row 2 in sharded mode: a halo-1 partition built from its pair's two
    shards is pending until grappa_halo_exchange ships the halo rows' features, global degrees and
    labels from their chunks' owners (here a 1-rank communicator's self transfers, or the local
    path without one); afterwards it is bitwise the replicated halo-1 partition and the oracle's
    halo sets and CSR"""
    uid = G.Context.nccl_unique_id() if nccl else None
    ctx = G.Context(0, rank=0, nranks=1, nccl_uid=uid) if nccl else G.Context(0)
    ds = prod
    C = 8
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rp, col, x, y, tr = upload(ds, tdt)
    ch, sh = shards_of(G, ctx, ds, C, dtype)
    chunk_of = Po.make_chunks(ds.wl.n, C, gen.seed_of("chunks"))
    for b, s in [(0, 3), (5, 2)]:
        p = G.grappa_repartition_shards(ctx, sh[b], sh[s], ch, C, halo=True)
        assert p.n_halo > 0
        with pytest.raises(G.GrappaError, match="pending"):
            h = torch.zeros(p.n_core, 16, device="cuda")
            ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
            G.grappa_layer_fwd_ex(ctx, p, "gcn", 16, 16, True, h, torch.zeros(16, 16, device="cuda"), h.clone(),
                                  None, ws, "f32", 0)
        G.grappa_halo_exchange(ctx, p, [sh[c] for c in range(C)], [0] * C, ch, C)
        one = G.grappa_repartition(ctx, rp, col, x, dtype, ch, C, b, s, tr, y, halo=True)
        torch.cuda.synchronize()
        for k in ("rowptr", "col", "core_global", "d_l", "d_g", "norm_gcn", "norm_sage", "seeds", "labels",
                  "node_w", "t_rowptr", "t_col"):
            assert torch.equal(getattr(p, k), getattr(one, k)), k
        assert torch.equal(p.x.view(torch.int16) if dtype == "bf16" else p.x,
                           one.x.view(torch.int16) if dtype == "bf16" else one.x)
        ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train, halo=True)
        assert np.array_equal(p.core_global.cpu().numpy(), ref["core"])
        assert np.array_equal(p.col.cpu().numpy(), ref["col"])
        assert np.array_equal(p.d_g.cpu().numpy(), ref["d_g"])
    q = G.grappa_repartition_shards(ctx, sh[0], sh[1], ch, C, halo=True)
    if nccl:
        # a shard this rank does not own is refused before anything moves
        with pytest.raises(G.GrappaError, match="E_ARG"):
            G.grappa_halo_exchange(ctx, q, [sh[2]], [0, 0, 1] + [0] * (C - 3), ch, C)
    # an owner that does not hold the requested rows: reported (on every rank), the partition
    # stays pending
    with pytest.raises(G.GrappaError, match="not in its owner"):
        G.grappa_halo_exchange(ctx, q, [sh[0], sh[1]], [0] * C, ch, C)
    with pytest.raises(G.GrappaError, match="pending"):
        h = torch.zeros(q.n_core, 16, device="cuda")
        G.grappa_layer_fwd_ex(ctx, q, "gcn", 16, 16, True, h, torch.zeros(16, 16, device="cuda"), h.clone(),
                              None, torch.empty(1 << 20, dtype=torch.uint8, device="cuda"), "f32", 0)
    ctx.check()
    ctx.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_sharded_halo_training_equals_replicated(G, prod, dtype):
    """sharded halo-1 training (owned shards only; halo features exchanged at every switch)
    reproduces the replicated halo-1 trainer's theta bit for bit over two switches"""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda sharded: Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                                 gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=1,
                                 dtype=dtype, sharded=sharded, halo=True)
    a, b = mk(False), mk(True)
    assert b.rowptr is None
    for _ in range(2):
        a.run_epoch()
        b.run_epoch()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(a.theta, b.theta)
    assert a.losses == b.losses
    ctx.close()
