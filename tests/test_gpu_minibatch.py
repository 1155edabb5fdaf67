"""GPU parity of a10 (isolated mini-batch sampling + SAGE mini-batch step) vs the oracle.

Bit-exact: the epoch seed order, every block (targets, sources, CSR, transpose).  1e-12: the
batch coverage factors.  1e-4 (fp32) / 2e-2 (bf16): the mini-batch gradient, with the ReLU
decisions the kernels took (R16b)."""
import math

import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import sampler as Sa

from _parity import assert_flips_bounded  # noqa: E402

pytestmark = pytest.mark.gpu
FAN = [6, 4, 3]        # input -> output layer (scaled-down {15, 10, 5})


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


@pytest.fixture(scope="module")
def setup(G):
    ctx = G.Context(0)
    wl = gen.small_workload("arxiv", n=12007, scale=14, num_samples=90_000, train_frac=0.3)
    ds = gen.make_dataset(wl)
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    ch = torch.empty(wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, wl.n, 4, gen.seed_of("chunks"), ch)
    chunk_of = Po.make_chunks(wl.n, 4, gen.seed_of("chunks"))
    ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, 1, 3, ds.train)
    parts = {}
    for dt in ("f32", "bf16"):
        x = torch.from_numpy(ds.x).to(d)
        x = x.to(torch.bfloat16) if dt == "bf16" else x
        parts[dt] = G.grappa_repartition(ctx, rp, col, x, dt, ch, 4, 1, 3, torch.from_numpy(ds.train).to(d),
                                         torch.from_numpy(ds.y).to(d))
    yield ctx, wl, ds, ref, parts
    ctx.close()


def test_epoch_order_bitexact(G, setup):
    ctx, wl, ds, ref, parts = setup
    p = parts["f32"]
    for epoch in (0, 3):
        order = torch.empty(p.n_seeds, dtype=torch.int32, device="cuda")
        G.grappa_epoch_seeds(ctx, p, 77, epoch, order)
        exp = np.concatenate(Sa.epoch_batches(ref, 77, epoch, 1000))
        assert np.array_equal(order.cpu().numpy(), exp)


@pytest.mark.parametrize("batch_index,fan", [(0, FAN), (5, FAN),
                                             (2, [25, 10]),            # P:489 2-layer fanouts
                                             (3, [20, 15, 10, 5]),     # P:489 4-layer fanouts
                                             (1, [32, 17])])           # the cap; the <=32 kernels
def test_sampled_blocks_bitexact(G, setup, batch_index, fan):
    ctx, wl, ds, ref, parts = setup
    p = parts["f32"]
    seeds = Sa.epoch_batches(ref, 9, 1, 300)[batch_index]
    b = G.grappa_sample(ctx, p, torch.from_numpy(seeds.astype(np.int32)).cuda(), fan, 9, 1, batch_index)
    blocks = Sa.sample_batch(ref, seeds, fan, 9, 1, batch_index)
    assert len(blocks) == len(fan) == len(b.blocks)
    for l, (gb, ob) in enumerate(zip(b.blocks, blocks)):
        assert gb["n_dst"] == ob["n_dst"] and gb["n_src"] == ob["n_src"], l
        assert np.array_equal(gb["src"].cpu().numpy(), ob["src"]), l
        assert np.array_equal(gb["rowptr"].cpu().numpy(), ob["rowptr"]), l
        assert np.array_equal(gb["col"].cpu().numpy(), ob["col"]), l
        # transpose = the same edge set grouped by source, targets ascending
        rows = np.repeat(np.arange(ob["n_dst"]), np.diff(ob["rowptr"]))
        o = np.lexsort((rows, ob["col"]))
        t_rp = np.searchsorted(ob["col"][o], np.arange(ob["n_src"] + 1))
        assert np.array_equal(gb["t_rowptr"].cpu().numpy(), t_rp), l
        assert np.array_equal(gb["t_col"].cpu().numpy(), rows[o]), l
        cnt = np.diff(ob["rowptr"])
        assert np.array_equal(gb["inv_cnt"].cpu().numpy(),
                              np.where(cnt > 0, 1.0 / np.maximum(cnt, 1), 0).astype(np.float32))
    d_l, d_g, s = Sa.batch_stats(ref, blocks)
    assert math.isclose(b.factors["uniform"], Co.c_uniform(d_l, d_g), rel_tol=1e-12)
    assert math.isclose(b.factors["resampling"], Co.c_resampling(d_l, d_g, s), rel_tol=1e-12)
    assert math.isclose(b.factors["resampling_hm"], Co.c_resampling_hm(d_l, d_g, s), rel_tol=1e-12)


def test_fanout_cap_rejected(G, setup):
    ctx, wl, ds, ref, parts = setup
    seeds = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception, match="fanout"):
        G.grappa_sample(ctx, parts["f32"], seeds, [33, 5], 9, 1, 0)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_minibatch_step_parity(G, setup, dtype):
    ctx, wl, ds, ref, parts = setup
    p = parts[dtype]
    seeds = Sa.epoch_batches(ref, 4, 0, 400)[1]
    b = G.grappa_sample(ctx, p, torch.from_numpy(seeds.astype(np.int32)).cuda(), FAN, 4, 0, 1)
    spec_dims, dp = wl.dims, wl.dims_pad
    theta = torch.cat([torch.from_numpy(np.concatenate(ws, 0).ravel()) for ws in ds.weights]).cuda()
    grad = torch.zeros_like(theta)
    ws = torch.empty(G.minibatch_ws_bytes(b, dp, dtype), dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    hidden = [torch.empty(b.blocks[l]["n_dst"], dp[l + 1], dtype=tdt, device="cuda") for l in range(2)]
    G.grappa_minibatch_step(ctx, p, b, dp, wl.K, theta, grad, ws, loss, dtype, hidden_out=hidden)
    torch.cuda.synchronize()
    blocks = Sa.sample_batch(ref, seeds, FAN, 4, 0, 1)
    W = [[np.asarray(w, np.float64) for w in ws_] for ws_ in ds.weights]      # padded blocks
    X = ds.x.astype(np.float64)[ref["core"]][blocks[0]["src"]]
    if dtype == "bf16":
        X = torch.from_numpy(ds.x).to(torch.bfloat16).float().numpy().astype(np.float64)[ref["core"]][blocks[0]["src"]]
    masks = [(h.float().cpu().numpy() > 0).astype(np.float64) for h in hidden]
    lg, cache = Sa.sage_forward(blocks, X, W, masks)
    assert_flips_bounded(cache, dtype, "minibatch step")
    K = wl.K
    L_ref, dZ = Mo.loss_and_dlogits(lg[:, :K], ds.y[ref["core"]][seeds], np.arange(len(seeds)))
    dZp = np.zeros_like(lg)
    dZp[:, :K] = dZ
    g_ref = Mo.flatten(Sa.sage_backward(blocks, cache, dZp, W))
    tol = 1e-4 if dtype == "f32" else 2e-2
    g = grad.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(g - g_ref)) / np.max(np.abs(g_ref)) <= tol
    assert math.isclose(loss.item(), L_ref, rel_tol=tol)


def test_minibatch_epoch_runs_and_reduces_loss(G, setup):
    """MinibatchTrainer (Alg. 1 lock-step over P = 4 partitions, M = 1): every iteration's
    aggregated update equals c_batch * g_batch and theta moves by -lr * that."""
    from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec
    ctx, wl, ds, ref, parts = setup
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    tr = MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 4,
                          gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=10,
                          fanouts=FAN, batch_size=500, sample_seed=3)
    th = [tr.theta.clone()]
    steps = []

    def grab():
        steps.append((tr.grad.clone(), tr.batch.factors["uniform"]))
        th.append(tr.theta.clone())

    tr.run_epoch(on_phase=grab)
    torch.cuda.synchronize()
    ctx.check()
    n_iter = sum(-(-p.n_seeds // 500) for p in tr.parts.values())
    assert len(steps) == n_iter
    for k, (g, c) in enumerate(steps):
        assert 0.0 < c <= 1.0
        d = (th[k] - th[k + 1]).double()
        ref = 0.05 * g.double()
        # theta is fp32 (~0.1): each update is exact up to theta's rounding (~1e-8)
        assert (d - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 2e-8


@pytest.mark.parametrize("fan", [[15, 10, 5], [1, 1, 2]])
def test_sampled_blocks_bitexact_hubs(G, fan):
    """Power-law partition with hub targets (d_l > 1024; the Floyd draw costs f per target
    whatever its degree): blocks bit-exact, at the paper's fanouts and at fanout 1."""
    ctx = G.Context(0)
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, train_frac=0.2)
    ds = gen.make_dataset(wl)
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    ch = torch.empty(wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, wl.n, 2, gen.seed_of("chunks"), ch)
    chunk_of = Po.make_chunks(wl.n, 2, gen.seed_of("chunks"))
    ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, 0, 1, ds.train)
    assert np.max(ref["d_l"]) > 1024
    p = G.grappa_repartition(ctx, rp, col, torch.from_numpy(ds.x).to(d), "f32", ch, 2, 0, 1,
                             torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d))
    hubs_seen = 0
    for bi in range(3):
        seeds = Sa.epoch_batches(ref, 11, 0, 1000)[bi]
        b = G.grappa_sample(ctx, p, torch.from_numpy(seeds.astype(np.int32)).cuda(), fan, 11, 0, bi)
        blocks = Sa.sample_batch(ref, seeds, fan, 11, 0, bi)
        for l, (gb, ob) in enumerate(zip(b.blocks, blocks)):
            hubs_seen += int(np.sum(np.asarray(ref["d_l"])[ob["dst"]] > 1024))
            assert np.array_equal(gb["src"].cpu().numpy(), ob["src"]), (bi, l)
            assert np.array_equal(gb["rowptr"].cpu().numpy(), ob["rowptr"]), (bi, l)
            assert np.array_equal(gb["col"].cpu().numpy(), ob["col"]), (bi, l)
    assert hubs_seen > 10
    ctx.close()


def test_sharded_minibatch_equals_replicated(G, setup):
    """sharded mode (a3 (i)) under the mini-batch trainer: partitions built from chunk shards
    feed the sampler exactly like replicated ones -- one epoch, theta bit for bit"""
    from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec
    ctx, wl, ds, ref, parts = setup
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    mk = lambda sh: MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 4,
                                     gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=10,
                                     fanouts=FAN, batch_size=500, sample_seed=3, dtype="bf16", sharded=sh)
    a, b = mk(False), mk(True)
    assert b.rowptr is None
    a.run_epoch()
    b.run_epoch()
    torch.cuda.synchronize()
    ctx.check()
    assert torch.equal(a.theta, b.theta)


def test_sampler_graph_replay_bitexact(G, setup):
    """grappa_sample_async on a side stream: the second call with a key captures the launch
    sequence into a CUDA graph and later calls replay it with new parameters (pinned params ->
    device).  Every call -- eager, capture, replays, and an eager call after a key change -- gives
    blocks bit-exact with a fresh eager sample and with the oracle."""
    ctx, wl, ds, ref, parts = setup
    p = parts["f32"]
    st = torch.cuda.Stream()
    order = Sa.epoch_batches(ref, 9, 1, 300)
    b = None
    fan_seq = [FAN, FAN, FAN, FAN, [5, 4, 3], FAN, FAN]
    for k, fan in enumerate(fan_seq):
        seeds = torch.from_numpy(order[k % len(order)].astype(np.int32)).cuda()
        l0 = ctx.launches()
        with torch.cuda.stream(st):
            b = G.grappa_sample_async(ctx, p, seeds, fan, 9, 1, k, b, stream=st)
        G.grappa_sample_wait(b)
        assert ctx.launches() > l0                   # replays count their captured launches
        fresh = G.grappa_sample(ctx, p, seeds, fan, 9, 1, k)
        blocks = Sa.sample_batch(ref, order[k % len(order)], fan, 9, 1, k)
        for l, (gb, fb, ob) in enumerate(zip(b.blocks, fresh.blocks, blocks)):
            for key in ("rowptr", "col", "t_rowptr", "t_col", "src", "inv_cnt"):
                assert torch.equal(gb[key], fb[key]), (k, l, key)
            assert np.array_equal(gb["col"].cpu().numpy(), ob["col"]), (k, l)
        assert b.factors == fresh.factors
