"""GPU parity of the node-level estimator (eq. (4)/(9) P:249-289, S:366-374,
reading R30) through the C ABI vs the f64 oracle.

Bars as DESIGN.md §5: bit-exact on the weights' integer inputs (d_l, d_g come from the
bit-exact repartition), 1e-6 relative on the fp32 weight rows, 1e-4 (fp32 storage) / 2e-2
(bf16) on activations, gradients and the aggregated update."""
import math

import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import sampler as Sa
from oracle import train as Tr

from _parity import assert_flips_bounded  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-4, "bf16": 2e-2}


def err(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)) if y.size else 0.0


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


@pytest.fixture(scope="module")
def ctx(G):
    c = G.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def prod():
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3)
    return gen.make_dataset(wl)


def _part(G, ctx, ds, C, b, s, dtype="f32"):
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    x = torch.from_numpy(ds.x).to(d)
    x = x.to(torch.bfloat16) if dtype == "bf16" else x
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    return G.grappa_repartition(ctx, rp, col, x, dtype, ch, C, b, s, torch.from_numpy(ds.train).to(d),
                                torch.from_numpy(ds.y).to(d))


def test_node_weight_rows(G, ctx, prod):
    part = _part(G, ctx, prod, 8, 2, 5)
    d_l, d_g = part.d_l.cpu().numpy(), part.d_g.cpu().numpy()
    w = Co.node_weights(d_l, d_g)
    nw = part.node_w.cpu().numpy().astype(np.float64)
    assert np.allclose(nw[0], w, rtol=1e-6, atol=0)
    assert np.allclose(nw[1], w / np.sqrt(d_l + 1.0), rtol=1e-6, atol=0)
    assert np.allclose(nw[2], np.where(d_l > 0, w / np.maximum(d_l, 1), 0.0), rtol=1e-6, atol=0)
    assert (w < 1).any() and (w == 1).any()


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("f_in,f_out", [(112, 128), (128, 48), (128, 128)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("normed", [False, True])
def test_layer_parity_node_level(G, ctx, prod, arch, f_in, f_out, dtype, normed):
    """layer-local parity of grappa_layer_fwd_ex / grappa_layer_bwd_ex with
    GRAPPA_LAYER_NODE_LEVEL against the oracle's weighted operator (GCN: also with both
    normalised-gradient flags, the chain the trainer uses)."""
    if normed and arch == "sage":
        pytest.skip("normalised gradients are GCN-only")
    part = _part(G, ctx, prod, 8, 2, 5, dtype)
    n = part.n_core
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in * 31 + f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    m = 1 if arch == "gcn" else 2
    w = (torch.randn(m * f_in, f_out, device="cuda", generator=g) / math.sqrt(f_in)).contiguous()
    h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
    saved = torch.empty(max(1, G.layer_saved_bytes(part, arch, f_in, f_out, dtype)), dtype=torch.uint8,
                        device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, arch, f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    NL = G.LAYER_NODE_LEVEL
    G.grappa_layer_fwd_ex(ctx, part, arch, f_in, f_out, True, h_in, w, h_out, saved, ws, dtype, NL)
    nrm = part.norm_gcn.double().cpu().numpy()
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-3)
    dz_k = (dz * part.norm_gcn[:, None]).to(tdt) if normed else dz.to(tdt)
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
    flags = NL | ((G.BWD_DZ_OUT_NORMED | G.BWD_DZ_IN_NORMED) if normed else 0)
    G.grappa_layer_bwd_ex(ctx, part, arch, f_in, f_out, True, dz_k, h_in, w, saved, dw, dz_in, ws, dtype,
                          flags)
    torch.cuda.synchronize()
    rp, cl = part.rowptr.cpu().numpy(), part.col.cpu().numpy()
    node_w = Co.node_weights(part.d_l.cpu().numpy(), part.d_g.cpu().numpy())
    op = Mo.operator(arch, rp, cl, n, node_w)
    H = _np(h_in)
    W = _np(w)
    Ws = [W] if arch == "gcn" else [W[:f_in], W[f_in:]]
    P, Z, Hn = Mo.layer_forward(arch, op, H, Ws, True)
    tol = TOL[dtype]
    assert err(_np(h_out), Hn) <= tol
    # the weighting is visible: the uncorrected operator is off by more than the tolerance
    _, _, H0 = Mo.layer_forward(arch, Mo.operator(arch, rp, cl, n), H, Ws, True)
    assert err(_np(h_out), H0) > 2 * tol
    dz_ref = _np(dz_k) / nrm[:, None] if normed else _np(dz_k)
    grads, dH = Mo.layer_backward(arch, op, H, P, Ws, dz_ref)
    assert err(_np(dw), np.concatenate(grads, axis=0)) <= tol
    ref_in = dH * (H > 0)
    if normed:
        ref_in = nrm[:, None] * ref_in
    assert err(_np(dz_in), ref_in) <= tol


def test_layer_flags_validated(G, ctx, prod):
    part = _part(G, ctx, prod, 8, 2, 5)
    n = part.n_core
    h = torch.zeros(n, 16, device="cuda")
    w = torch.zeros(16, 16, device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, "gcn", 16, 16, "f32"), dtype=torch.uint8, device="cuda")
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_fwd_ex(ctx, part, "gcn", 16, 16, True, h, w, h.clone(), None, ws, "f32", 8)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_bwd_ex(ctx, part, "gcn", 16, 16, True, h, h, w, None, w.clone(), h.clone(), ws,
                              "f32", 16)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_epoch_parity_node_level(G, ctx, prod, dtype):
    """Alg. 1 over P = 8 partitions (M = 1, repartition every epoch) with corr "node": every
    phase's aggregated update vs the oracle's node-level gradient at the GPU's own theta (the
    kernels' ReLU decisions, R16b), then the first epoch's theta trajectory (fp32)."""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    lr = 0.05
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr="node", lr=lr, repartition_every=1, dtype=dtype)
    ghat, thetas, masks = [], [], []

    def snap():
        sp = tr.spec
        mats, off = [], 0
        for l, (a, b) in enumerate(sp.layer_shapes()):
            blk = tr.theta[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
            gb = tr.grad[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
            off += a * b
            mats.append(([blk[:sp.dims[l], :sp.dims[l + 1]]], [gb[:sp.dims[l], :sp.dims[l + 1]]]))
        return Mo.flatten([m[0] for m in mats]), Mo.flatten([m[1] for m in mats])

    thetas.append(snap()[0])

    def grab():
        th, gh = snap()
        ghat.append(gh)
        thetas.append(th)
        n = tr.parts[len(masks) % wl.chunks].n_core
        masks.append([(tr.H[l][:n, :wl.dims[l]].float() > 0).cpu().numpy().astype(np.float64)
                      for l in range(1, wl.depth)])

    tr.run_epoch(on_phase=grab)
    torch.cuda.synchronize()
    ctx.check()
    P = wl.chunks
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    sched = Po.sweep_schedule(P, P)
    X = ds.x[:, :wl.F].astype(np.float64)
    if dtype == "bf16":
        X = torch.from_numpy(ds.x[:, :wl.F]).to(torch.bfloat16).double().numpy()
    Wref = [[np.asarray(w, np.float64)[:wl.dims[l], :wl.dims[l + 1]] for w in ws]
            for l, ws in enumerate(ds.weights)]
    shapes = [[w.shape for w in ws] for ws in Wref]
    for k in range(P):
        b, s = sched[0][k]
        part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
        nw = Co.node_weights(part["d_l"], part["d_g"])
        _, g, _, cache = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                                Mo.unflatten(thetas[k], shapes), masks[k], node_w=nw)
        assert_flips_bounded(cache, dtype, f"node-level phase {k}")
        # the node-level gradient differs from the uncorrected one (the weights act)
        _, g0, _, _ = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                             Mo.unflatten(thetas[k], shapes))      # uncorrected, own ReLU
        assert err(g0, g) > 1e-3
        assert err(ghat[k], Co.aggregate([1.0], [g], 1)) <= TOL[dtype], k
    if dtype == "f32":
        final, _ = Tr.run(wl.arch, ds.rowptr, ds.col, X, ds.y, ds.train, Wref, chunk_of, P, P, 1,
                          "node", lr, 1, 1)
        assert err(thetas[P], Mo.flatten(final)) <= 1e-4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_minibatch_node_level(G, ctx, dtype):
    """SAGE mini-batch step with GRAPPA_LAYER_NODE_LEVEL: inv_cnt_node = (d_l/d_g)/|S(v)| and the
    gradient vs the oracle's weighted block operators."""
    wl = gen.small_workload("arxiv", n=12007, scale=14, num_samples=90_000, train_frac=0.3)
    ds = gen.make_dataset(wl)
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    ch = torch.empty(wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, wl.n, 4, gen.seed_of("chunks"), ch)
    chunk_of = Po.make_chunks(wl.n, 4, gen.seed_of("chunks"))
    ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, 1, 3, ds.train)
    x = torch.from_numpy(ds.x).to(d)
    x = x.to(torch.bfloat16) if dtype == "bf16" else x
    p = G.grappa_repartition(ctx, rp, col, x, dtype, ch, 4, 1, 3, torch.from_numpy(ds.train).to(d),
                             torch.from_numpy(ds.y).to(d))
    FAN = [6, 4, 3]
    seeds = Sa.epoch_batches(ref, 4, 0, 400)[1]
    b = G.grappa_sample(ctx, p, torch.from_numpy(seeds.astype(np.int32)).cuda(), FAN, 4, 0, 1)
    blocks = Sa.sample_batch(ref, seeds, FAN, 4, 0, 1)
    node_w = Co.node_weights(ref["d_l"], ref["d_g"])
    for gb, ob in zip(b.blocks, blocks):
        cnt = np.diff(ob["rowptr"])
        exp = np.where(cnt > 0, node_w[ob["dst"]] / np.maximum(cnt, 1), 0.0)
        assert np.allclose(gb["inv_cnt_node"].cpu().numpy(), exp, rtol=1e-6, atol=0)
    dp = wl.dims_pad
    theta = torch.cat([torch.from_numpy(np.concatenate(ws, 0).ravel()) for ws in ds.weights]).cuda()
    grad = torch.zeros_like(theta)
    ws = torch.empty(G.minibatch_ws_bytes(b, dp, dtype), dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    hidden = [torch.empty(b.blocks[l]["n_dst"], dp[l + 1], dtype=tdt, device="cuda") for l in range(2)]
    G.grappa_minibatch_step(ctx, p, b, dp, wl.K, theta, grad, ws, loss, dtype, hidden_out=hidden,
                            flags=G.LAYER_NODE_LEVEL)
    torch.cuda.synchronize()
    W = [[np.asarray(w, np.float64) for w in ws_] for ws_ in ds.weights]
    xs = ds.x.astype(np.float64)
    if dtype == "bf16":
        xs = torch.from_numpy(ds.x).to(torch.bfloat16).double().numpy()
    X = xs[ref["core"]][blocks[0]["src"]]
    masks = [(h.float().cpu().numpy() > 0).astype(np.float64) for h in hidden]
    lg, cache = Sa.sage_forward(blocks, X, W, masks, node_w=node_w)
    assert_flips_bounded(cache, dtype, "node-level minibatch step")
    K = wl.K
    L_ref, dZ = Mo.loss_and_dlogits(lg[:, :K], ds.y[ref["core"]][seeds], np.arange(len(seeds)))
    dZp = np.zeros_like(lg)
    dZp[:, :K] = dZ
    g_ref = Mo.flatten(Sa.sage_backward(blocks, cache, dZp, W))
    g = grad.cpu().numpy().astype(np.float64)
    assert err(g, g_ref) <= TOL[dtype]
    assert math.isclose(loss.item(), L_ref, rel_tol=TOL[dtype])
    assert b.factors["node"] == 1.0


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("node", [False, True])
@pytest.mark.parametrize("f_in,f_out", [(112, 128), (16, 48)])
def test_gcn_input_layer_aggregate_first(G, ctx, prod, dtype, node, f_in, f_out):
    """GRAPPA_LAYER_INPUT (GCN): Z = (Ahat h_in) W with P kept in `saved`; backward dW = P^T dz
    only (no dh_in).  Same operator as the transform-first layer (R29 re-association)."""
    part = _part(G, ctx, prod, 8, 2, 5, dtype)
    n = part.n_core
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in + f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).to(tdt)
    w = (torch.randn(f_in, f_out, device="cuda", generator=g) / math.sqrt(f_in)).contiguous()
    fl = G.LAYER_INPUT | (G.LAYER_NODE_LEVEL if node else 0)
    saved = torch.empty(G.layer_saved_bytes(part, "gcn", f_in, f_out, dtype, fl), dtype=torch.uint8, device="cuda")
    assert saved.numel() == n * f_in * (2 if dtype == "bf16" else 4)
    ws = torch.empty(G.layer_ws_bytes(part, "gcn", f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
    G.grappa_layer_fwd_ex(ctx, part, "gcn", f_in, f_out, True, h_in, w, h_out, saved, ws, dtype, fl)
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-3).to(tdt)
    dw = torch.empty_like(w)
    G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, f_out, False, dz, h_in, w, saved, dw, None, ws, dtype, fl)
    torch.cuda.synchronize()
    node_w = Co.node_weights(part.d_l.cpu().numpy(), part.d_g.cpu().numpy()) if node else None
    op = Mo.operator("gcn", part.rowptr.cpu().numpy(), part.col.cpu().numpy(), n, node_w)
    H, W = _np(h_in), _np(w)
    P, Z, Hn = Mo.layer_forward("gcn", op, H, [W], True)
    tol = TOL[dtype]
    assert err(_np(h_out), Hn) <= tol
    grads, _ = Mo.layer_backward("gcn", op, H, P, [W], _np(dz))
    assert err(_np(dw), grads[0]) <= tol
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, f_out, False, dz, h_in, w, saved, dw,
                              torch.empty(n, f_in, device="cuda", dtype=tdt), ws, dtype, fl)
