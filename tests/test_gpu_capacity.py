"""Capacity mode (Alg. 1 with partitions streamed from host memory, P:395,
P:139): partition images round-trip bit-exactly (grappa_part_save / grappa_part_load),
and an epoch that streams every phase's partition from pinned host memory into two device slots
reproduces the resident-partition epoch bit for bit (same kernels, same inputs, same order); so does
capacity mode from chunk shards (host shard images, partitions extracted per phase on the device).
"""
import pytest
import torch

import gen

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


@pytest.mark.parametrize("halo", [False, True])
def test_image_roundtrip(G, prod, halo):
    ctx = G.Context(0)
    ds = prod
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, ds.wl.n, 8, gen.seed_of("chunks"), ch)
    p = G.grappa_repartition(ctx, rp, col, torch.from_numpy(ds.x).to(d).to(torch.bfloat16), "bf16", ch, 8, 1, 6,
                             torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d), halo=halo)
    host = torch.empty(p.image_bytes(), dtype=torch.uint8, pin_memory=True)
    p.save(host)
    torch.cuda.synchronize()
    info = G.Part.image_info(host)
    assert info.n_core == p.n_core and info.nnz == p.nnz and info.n_halo == p.n_halo
    q = G.Part().load_image(host)
    torch.cuda.synchronize()
    for k in ("rowptr", "col", "core_global", "d_l", "d_g", "norm_gcn", "norm_sage", "seeds", "labels",
              "node_w"):
        assert torch.equal(getattr(p, k), getattr(q, k)), k
    assert torch.equal(p.x.view(torch.int16), q.x.view(torch.int16))
    if halo:
        assert torch.equal(p.t_rowptr, q.t_rowptr) and torch.equal(p.t_col, q.t_col)
    assert q.info.c_resampling == p.info.c_resampling and q.info.n_slots == p.info.n_slots
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.Part().load_image(torch.zeros(4096, dtype=torch.uint8, pin_memory=True))
    ctx.close()


@pytest.mark.parametrize("halo,dtype,cap", [(False, "bf16", True), (True, "f32", True),
                                            (False, "bf16", "shards"), (False, "f32", "shards")])
def test_capacity_epoch_equals_resident(G, prod, halo, dtype, cap):
    """cap=True: partition images; cap="shards": chunk-shard images in host memory, the partition
    extracted per phase from its pair's two shards (the device never holds the global graph)"""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda cap: Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                             gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=1,
                             dtype=dtype, halo=halo, capacity=cap)
    a, b = mk(False), mk(cap)
    if cap == "shards":
        assert b.rowptr is None and b.col is None and b.x is None       # no global array on the device
    for _ in range(2):                       # two super-epochs (repartition every epoch)
        a.run_epoch()
        b.run_epoch()
    torch.cuda.synchronize()
    ctx.check()
    assert not b.parts or len(b.parts) == 1
    assert torch.equal(a.theta, b.theta)
    assert not torch.equal(a.theta, mk(False).theta)       # the epochs did move theta
    ctx.close()


@pytest.mark.parametrize("dtype,eager_min", [("bf16", None), ("f32", None), ("bf16", 0)])
def test_graph_epochs_equal_eager(G, prod, dtype, eager_min):
    """CUDA-graph replay (run_epoch_graph: the first epoch of a super-epoch runs eagerly while the
    same launches are captured, later epochs replay) reproduces eager epochs bit for bit, across
    a super-epoch switch"""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda: Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                         gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=2, dtype=dtype)
    a, b = mk(), mk()
    if eager_min is not None:                # the eager-while-capturing path of large partitions
        b.graph_eager_min_nnz = eager_min
    for _ in range(5):                       # super-epochs 1, 1, 2, 2, 3
        a.run_epoch()
        b.run_epoch_graph()
    torch.cuda.synchronize()
    ctx.check()
    assert b.graph is not None and b.graph_launches > 0
    assert torch.equal(a.theta, b.theta)
    assert a.losses == b.losses if hasattr(a, "losses") else True
    ctx.close()


@pytest.mark.parametrize("use_graph", [False, True])
def test_e2e_epochs_equal_resident(G, prod, use_graph):
    """bench.measure_e2e (the end-to-end number: every partition uploaded from pinned host images
    each epoch, the first phase's partition during the previous epoch, the loss read back; with
    use_graph the epochs are graph replays and switches are prefetched) trains exactly what the
    device-resident loop trains: theta bitwise equal after 1 + K epochs across super-epoch
    switches"""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda: Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                         gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=2, dtype="bf16")
    a, b = mk(), mk()
    stream = torch.cuda.current_stream()
    K = 5
    r = bench.measure_e2e(a, stream, K, torch.cuda.synchronize, 1, None, ds.nnz, use_graph=use_graph)
    assert r["h2d_bytes_per_step"] > 0
    b.epoch = 2                                  # measure_e2e starts on the next boundary
    for _ in range(1 + K):
        b.run_epoch()
    torch.cuda.synchronize()
    ctx.check()
    assert a.epoch == b.epoch
    assert torch.equal(a.theta, b.theta)
    ctx.close()
