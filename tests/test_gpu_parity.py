"""GPU parity: the CUDA path through the C ABI vs the f64 oracle on the same seeded inputs.

Bars: bit-exact on chunking, induced CSR, degrees, seeds, D and c_resampling;
1e-12 relative on c_uniform / c_resampling_hm; err = max|x-y| / max|y| <= 1e-4 (fp32 storage)
or 2e-2 (bf16 storage) on activations, gradients and the aggregated update.
"""
import math

import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import train as Tr

from _parity import assert_flips_bounded  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def err(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)) if y.size else 0.0


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


def small_products():
    # products generator at ~1/120 scale: RMAT hubs well above the 256-edge split length
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3)
    return gen.make_dataset(wl)


def small_arxiv():
    wl = gen.small_workload("arxiv", n=12007, scale=14, num_samples=90_000)
    return gen.make_dataset(wl)


@pytest.fixture(scope="module")
def prod():
    return small_products()


@pytest.fixture(scope="module")
def arxiv():
    return small_arxiv()


def upload(ds):
    d = "cuda"
    return (torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d),
            torch.from_numpy(ds.x).to(d), torch.from_numpy(ds.y).to(d),
            torch.from_numpy(ds.train).to(d))


# ----------------------------------------------------------------------------- a1
@pytest.mark.parametrize("n,C", [(2, 2), (17, 3), (2708, 4), (20011, 8), (1_000_003, 8), (4097, 4097)])
def test_partition_bitexact(G, ctx, n, C):
    seed = gen.seed_of("chunks")
    ch = torch.empty(n, dtype=torch.int32, device="cuda")
    sizes = G.grappa_partition(ctx, n, C, seed, ch)
    ref = Po.make_chunks(n, C, seed)
    assert np.array_equal(ch.cpu().numpy(), ref)
    assert sizes == np.bincount(ref, minlength=C).tolist()


def test_partition_errors(G, ctx):
    ch = torch.empty(10, dtype=torch.int32, device="cuda")
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_partition(ctx, 10, 1, 0, ch)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_partition(ctx, 10, 11, 0, ch)


# ----------------------------------------------------------------------------- a3
@pytest.mark.parametrize("C,pairs", [(8, [(0, 1), (3, 7), (6, 2)]), (2, [(0, 1)]), (4, [(1, 3)])])
def test_repartition_bitexact(G, ctx, prod, C, pairs):
    ds = prod
    rp, col, x, y, tr = upload(ds)
    seed = gen.seed_of("chunks")
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device="cuda")
    G.grappa_partition(ctx, ds.wl.n, C, seed, ch)
    chunk_of = Po.make_chunks(ds.wl.n, C, seed)
    part = None
    for b, s in pairs:
        part = G.grappa_repartition(ctx, rp, col, x, "f32", ch, C, b, s, tr, y, part)
        ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
        assert np.array_equal(part.core_global.cpu().numpy(), ref["core"])
        assert np.array_equal(part.rowptr.cpu().numpy(), ref["rowptr"])
        assert np.array_equal(part.col.cpu().numpy(), ref["col"])
        assert np.array_equal(part.d_l.cpu().numpy(), ref["d_l"])
        assert np.array_equal(part.d_g.cpu().numpy(), ref["d_g"])
        assert np.array_equal(part.seeds.cpu().numpy(), ref["seeds"])
        assert np.array_equal(part.labels.cpu().numpy(), ds.y[ref["core"]])
        assert np.array_equal(part.x.cpu().numpy(), ds.x[ref["core"]])
        s_dl, s_dg = ref["d_l"][ref["seeds"]], ref["d_g"][ref["seeds"]]
        assert part.info.D == int(np.sum((s_dg - s_dl)[s_dl > 0]))
        assert part.info.c_resampling == Co.c_resampling(s_dl, s_dg)          # bit-exact
        assert math.isclose(part.info.c_uniform, Co.c_uniform(s_dl, s_dg), rel_tol=1e-12)
        assert math.isclose(part.info.c_resampling_hm, Co.c_resampling_hm(s_dl, s_dg), rel_tol=1e-12)
        nrm = part.norm_gcn.cpu().numpy()
        assert np.array_equal(nrm, (1.0 / np.sqrt(ref["d_l"] + 1.0)).astype(np.float32))
        if C == 2:
            assert np.array_equal(ref["d_l"], ref["d_g"]) and part.info.c_resampling == 1.0
        assert part.info.n_heavy == int(np.sum(ref["d_l"] > 256))


def test_repartition_errors(G, ctx, prod):
    rp, col, x, y, tr = upload(prod)
    ch = torch.empty(prod.wl.n, dtype=torch.int32, device="cuda")
    G.grappa_partition(ctx, prod.wl.n, 4, 1, ch)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_repartition(ctx, rp, col, x, "f32", ch, 4, 2, 2, tr, y)
    with pytest.raises(G.GrappaError, match="E_EMPTY"):
        G.grappa_repartition(ctx, rp, col, x, "f32", ch, 4, 0, 1, torch.zeros_like(tr), y)


# ----------------------------------------------------------------------------- a4-a6
def _part(G, ctx, ds, C, b, s, dtype="f32"):
    rp, col, x, y, tr = upload(ds)
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device="cuda")
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    xt = x.to(torch.bfloat16) if dtype == "bf16" else x
    return G.grappa_repartition(ctx, rp, col, xt, dtype, ch, C, b, s, tr, y)


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("f_in,f_out", [(112, 128), (128, 48), (128, 16), (16, 128), (256, 256),
                                         (112, 256), (256, 48),
                                         (1440, 128), (1440, 16)])   # cora's input layer: streamed weights
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layer_parity(G, ctx, prod, arch, f_in, f_out, dtype):
    """Layer-local parity: the oracle sees the GPU's own (upcast) layer inputs."""
    part = _part(G, ctx, prod, 8, 2, 5, dtype)
    n = part.n_core
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in * 1000 + f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    m = 1 if arch == "gcn" else 2
    w = (torch.randn(m * f_in, f_out, device="cuda", generator=g) / math.sqrt(f_in)).contiguous()
    h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
    saved = torch.empty(max(1, G.layer_saved_bytes(part, arch, f_in, f_out, dtype)), dtype=torch.uint8, device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, arch, f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    G.grappa_layer_fwd(ctx, part, arch, f_in, f_out, True, h_in, w, h_out, saved, ws, dtype)
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-3).to(tdt)
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
    G.grappa_layer_bwd(ctx, part, arch, f_in, f_out, True, dz, h_in, w, saved, dw, dz_in, ws, dtype)
    torch.cuda.synchronize()
    rp, cl = part.rowptr.cpu().numpy(), part.col.cpu().numpy()
    op = Mo.operator(arch, rp, cl, n)
    H = _np(h_in)
    W = _np(w)
    Ws = [W] if arch == "gcn" else [W[:f_in], W[f_in:]]
    P, Z, Hn = Mo.layer_forward(arch, op, H, Ws, True)
    tol = TOL[dtype]
    assert err(_np(h_out), Hn) <= tol
    grads, dH = Mo.layer_backward(arch, op, H, P, Ws, _np(dz))
    dW_ref = np.concatenate(grads, axis=0)
    assert err(_np(dw), dW_ref) <= tol
    ref_in = dH * (H > 0)
    assert err(_np(dz_in), ref_in) <= tol


@pytest.mark.parametrize("f_in,f_out", [(112, 128), (128, 48), (128, 128)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layer_bwd_normalised_flags(G, ctx, prod, f_in, f_out, dtype):
    """grappa_layer_bwd_ex with both GCN normalised-gradient flags (reading R29): the kernel
    gets dz' = N dz and must return dW and N dz_in of the oracle's backward for dz = dz'/N."""
    part = _part(G, ctx, prod, 8, 2, 5, dtype)
    n = part.n_core
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in + 7 * f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    w = (torch.randn(f_in, f_out, device="cuda", generator=g) / math.sqrt(f_in)).contiguous()
    nrm = part.norm_gcn
    dz_s = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-3 * nrm[:, None]).to(tdt)
    saved = torch.empty(1, dtype=torch.uint8, device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, "gcn", f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
    G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, f_out, True, dz_s, h_in, w, saved, dw, dz_in, ws, dtype,
                          G.BWD_DZ_OUT_NORMED | G.BWD_DZ_IN_NORMED)
    torch.cuda.synchronize()
    N = nrm.cpu().numpy().astype(np.float64)
    op = Mo.operator("gcn", part.rowptr.cpu().numpy(), part.col.cpu().numpy(), n)
    H = _np(h_in)
    Ws = [_np(w)]
    P, Z, _ = Mo.layer_forward("gcn", op, H, Ws, True)
    grads, dH = Mo.layer_backward("gcn", op, H, P, Ws, _np(dz_s) / N[:, None])
    tol = TOL[dtype]
    assert err(_np(dw), grads[0]) <= tol
    assert err(_np(dz_in), N[:, None] * dH * (H > 0)) <= tol
    # flags are GCN-only and must be known
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, f_out, True, dz_s, h_in, w, saved, dw, dz_in, ws,
                              dtype, 8)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_bwd_ex(ctx, part, "sage", f_in, f_out, True, dz_s, h_in, w, saved, dw, dz_in, ws,
                              dtype, 1)


@pytest.mark.parametrize("which,K,kpad", [("prod", 47, 48), ("arxiv", 40, 48)])
def test_loss_parity(G, ctx, prod, arxiv, which, K, kpad):
    ds = prod if which == "prod" else arxiv
    part = _part(G, ctx, ds, 8, 1, 4)
    n = part.n_core
    g = torch.Generator(device="cuda").manual_seed(K)
    logits = torch.randn(n, kpad, device="cuda", generator=g) * 3
    logits[:, K:] = 0
    dl = torch.empty_like(logits)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    G.grappa_loss(ctx, part, logits, K, kpad, dl, loss, "f32")
    torch.cuda.synchronize()
    ref_loss, ref_dz = Mo.loss_and_dlogits(_np(logits)[:, :K], part.labels.cpu().numpy(),
                                           part.seeds.cpu().numpy())
    assert math.isclose(loss.item(), ref_loss, rel_tol=1e-5)
    assert err(_np(dl)[:, :K], ref_dz) <= 1e-4
    assert np.all(_np(dl)[:, K:] == 0)


# ----------------------------------------------------------------------------- end to end
def _oracle_weights(ds, spec_dims):
    """padded per-layer GPU blocks -> logical f64 blocks for the oracle"""
    out = []
    for l, ws in enumerate(ds.weights):
        out.append([np.asarray(w, dtype=np.float64)[:spec_dims[l], :spec_dims[l + 1]] for w in ws])
    return out


def _logical(trainer, flat):
    """padded flat GPU layout (theta or grad) -> logical oracle layout"""
    sp = trainer.spec
    mats, off = [], 0
    for l, (a, b) in enumerate(sp.layer_shapes()):
        blk = flat[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
        off += a * b
        fi, fo, fip = sp.dims[l], sp.dims[l + 1], sp.dims_pad[l]
        if sp.arch == "gcn":
            mats.append([blk[:fi, :fo]])
        else:
            mats.append([blk[:fi, :fo], blk[fip:fip + fi, :fo]])
    return Mo.flatten(mats)


@pytest.mark.parametrize("which,corr,epochs,rep,capacity", [("prod", "resampling", 2, 1, False),
                                                            ("prod", "uniform", 1, 10, False),
                                                            ("arxiv", "resampling", 1, 10, False),
                                                            ("arxiv", "none", 2, 1, False),
                                                            ("prod", "uniform", 2, 1, True),
                                                            ("arxiv", "resampling_hm", 1, 10, True),
                                                            ("prod", "uniform", 2, 1, "shards"),
                                                            ("arxiv", "resampling", 1, 10, "shards")])
def test_epoch_parity(G, ctx, prod, arxiv, which, corr, epochs, rep, capacity):
    """Alg. 1 end to end on 1 GPU (P = 8 partitions, M = 1 per phase): theta after the run
    matches the oracle's phase loop.  lr is raised so the update is visible next to theta.
    capacity: partitions parked as host images and streamed into two device slots per phase
    (§8(f) row 3) -- the same oracle comparison, phase by phase."""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ds = prod if which == "prod" else arxiv
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    lr = 0.05
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr=corr, lr=lr, repartition_every=rep, capacity=capacity)
    ghat, thetas, masks = [], [_logical(tr, tr.theta)], []

    def grab():
        ghat.append(_logical(tr, tr.grad))
        thetas.append(_logical(tr, tr.theta))
        n = tr.parts[len(masks) % wl.chunks].n_core
        # the kernels' own ReLU decisions (fp32 pre-activation > 0), reading R16b
        masks.append([(tr.H[l][:n, :wl.dims[l]] > 0).cpu().numpy().astype(np.float64)
                      for l in range(1, wl.depth)])

    for _ in range(epochs):
        tr.run_epoch(on_phase=grab)
    torch.cuda.synchronize()
    ctx.check()
    P = wl.chunks
    assert len(ghat) == epochs * P
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    sched = Po.sweep_schedule(P, P)
    X = ds.x[:, :wl.F].astype(np.float64)
    Wref = _oracle_weights(ds, wl.dims)
    shapes = [[w.shape for w in ws] for ws in Wref]
    # step-local parity: the oracle's aggregated update at the GPU's own theta of each phase
    # (ReLU kinks make multi-step trajectories chaotic at the 1e-7 level, so every phase is
    # checked from the same starting point), with the ReLU decisions the kernels took
    for k in range(epochs * P):
        e, w = divmod(k, P)
        b, s = sched[(e // rep) % len(sched)][w]
        part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
        Wk = Mo.unflatten(thetas[k], shapes)
        _, g, _, cache = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                                Wk, masks[k])
        ref = Co.aggregate([Tr.partition_factor(corr, part)], [g], 1)
        assert err(ghat[k], ref) <= 1e-4, k
        # the decisions themselves: disagreements only where |Z| is at rounding level (R16b)
        assert_flips_bounded(cache, "f32", f"phase {k}")
        step = thetas[k] - thetas[k + 1]
        if corr != "resampling":                       # literal c_resampling ~1e-6: update < ulp
            assert err(step, lr * ghat[k]) <= 1e-3, k
    # trajectory over the first epoch (8 SGD steps) against the oracle's own phase loop
    final, recs = Tr.run(wl.arch, ds.rowptr, ds.col, X, ds.y, ds.train, Wref, chunk_of, P, P, 1,
                         corr, lr, 1, rep)
    assert err(thetas[P], Mo.flatten(final)) <= 1e-4


@pytest.mark.parametrize("arch,op,dtype,alt", [("gcn", "gemm", "bf16", 1), ("sage", "gemm", "bf16", 1),
                                               ("gcn", "gemm", "f32", 2), ("sage", "gemm", "f32", 2),
                                               ("gcn", "gemm", "f32", 1), ("sage", "gemm", "f32", 1),
                                               ("gcn", "spmm", "bf16", 1), ("sage", "spmm", "f32", 1),
                                               ("gcn", "spmm", "bf16", 3), ("gcn", "spmm", "bf16", 2),
                                               ("gcn", "spmm", "bf16", 5), ("sage", "spmm", "f32", 5),
                                               ("sage", "spmm", "bf16", 5), ("gcn", "wstream", "bf16", 2),
                                               ("sage", "wstream", "bf16", 2), ("gcn", "wstream", "bf16", 1)])
def test_kernel_variants_agree(G, ctx, prod, arch, op, dtype, alt):
    """Alternative implementations agree on the same layer and inputs: bf16 tcgen05 GEMMs vs
    the CUDA-core GEMMs; the split-fp32 tcgen05 GEMMs (fp32 storage) vs the FFMA ones (1e-5); the
    row-group SpMM vs the warp-per-row SpMM and its other schedules."""
    part = _part(G, ctx, prod, 8, 3, 6, dtype)
    n, f_in, f_out = part.n_core, 112, 48
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(7)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    m = 1 if arch == "gcn" else 2
    w = torch.randn(m * f_in, f_out, device="cuda", generator=g) / 10
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-2).to(tdt)
    outs = []
    default = 0
    for variant in (default, alt):
        ctx.set_variant(op, variant)
        h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
        saved = torch.empty(max(1, G.layer_saved_bytes(part, arch, f_in, f_out, dtype)), dtype=torch.uint8, device="cuda")
        ws = torch.empty(G.layer_ws_bytes(part, arch, f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
        G.grappa_layer_fwd(ctx, part, arch, f_in, f_out, True, h_in, w, h_out, saved, ws, dtype)
        dw = torch.empty_like(w)
        dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
        G.grappa_layer_bwd(ctx, part, arch, f_in, f_out, True, dz, h_in, w, saved, dw, dz_in, ws, dtype)
        torch.cuda.synchronize()
        outs.append((_np(h_out), _np(dw), _np(dz_in)))
    ctx.set_variant(op, default)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        ctx.set_variant("nope", 1)
    with pytest.raises(G.GrappaError, match="E_ARG"):
        ctx.set_variant(op, 7)
    for a, b in zip(*outs):
        assert err(a, b) <= (1e-2 if dtype == "bf16" else 1e-5)
    if (op == "spmm" and alt == 5) or op == "wstream":
        # same edges / same bf16 weight values and MMA order: bitwise equal
        # the lean unweighted gather walks the same edges in the same order: bitwise equal
        for a, b in zip(*outs):
            assert np.array_equal(a, b)


def test_loss_dz_normed_flag(G, ctx, prod):
    """grappa_loss_ex(GRAPPA_LOSS_DZ_NORMED): dZ rows scaled by norm_gcn (R29 chain), same loss."""
    part = _part(G, ctx, prod, 8, 1, 4)
    n = part.n_core
    g = torch.Generator(device="cuda").manual_seed(3)
    logits = torch.randn(n, 48, device="cuda", generator=g) * 3
    logits[:, 47:] = 0
    dl0, dl1 = torch.empty_like(logits), torch.empty_like(logits)
    l0 = torch.zeros(1, dtype=torch.float64, device="cuda")
    l1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    G.grappa_loss(ctx, part, logits, 47, 48, dl0, l0, "f32")
    G.grappa_loss(ctx, part, logits, 47, 48, dl1, l1, "f32", flags=1)
    torch.cuda.synchronize()
    assert l0.item() == l1.item()
    ref_loss, ref_dz = Mo.loss_and_dlogits(_np(logits)[:, :47], part.labels.cpu().numpy(), part.seeds.cpu().numpy())
    nrm = part.norm_gcn.cpu().numpy().astype(np.float64)
    assert err(_np(dl1)[:, :47], nrm[:, None] * ref_dz) <= 1e-4
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_loss(ctx, part, logits, 47, 48, dl1, l1, "f32", flags=2)


@pytest.mark.parametrize("f_in,f_out,normed,relu", [(128, 128, True, True), (128, 48, False, True),
                                                    (112, 128, True, False), (80, 16, False, True)])
def test_backward_pair_matches_separate_gemms(G, ctx, prod, f_in, f_out, normed, relu):
    """GCN backward: the one-pass pair kernel (dz_in and dW from one read of dT and h_in) gives
    the separate NN/TN kernels' dz_in bit for bit (same MMAs, same epilogue) and dW up to the
    fp32 summation order of the split (1e-5); the oracle parity of the layer is covered by
    test_layer_parity, which runs the pair by default"""
    part = _part(G, ctx, prod, 8, 3, 6, "bf16")
    n = part.n_core
    g = torch.Generator(device="cuda").manual_seed(f_in + 7 * f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(f_in, f_out, device="cuda", generator=g) / 10
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    outs = []
    flags = 3 if normed else 0
    for off in (0, 1):
        ctx.set_variant("pair", off)
        ws = torch.empty(G.layer_ws_bytes(part, "gcn", f_in, f_out, "bf16"), dtype=torch.uint8, device="cuda")
        dw = torch.full_like(w, float("nan"))
        dz_in = torch.empty(n, f_in, device="cuda", dtype=torch.bfloat16)
        G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, f_out, relu, dz, h_in, w, None, dw, dz_in, ws, "bf16",
                              flags=flags)
        torch.cuda.synchronize()
        outs.append((dz_in.clone(), dw.clone()))
    ctx.set_variant("pair", 0)
    (a_dz, a_dw), (b_dz, b_dw) = outs
    assert torch.equal(a_dz.view(torch.int16), b_dz.view(torch.int16))
    assert torch.isfinite(a_dw).all()
    assert err(_np(a_dw), _np(b_dw)) <= 1e-5


@pytest.mark.parametrize("eager_capture", [True, False])
def test_bf16_graph_epochs_vs_oracle(G, ctx, eager_capture):
    """The bench's launch configuration end to end against the oracle: products-shaped GCN-8
    (100 -> 128 x 7 -> 47), P = 8, M = 1, bf16 storage, epochs replayed from a CUDA graph per
    super-epoch (run_epoch_graph: eager-while-capturing, as the bench runs products, or
    record-then-replay), aggregate-first input layer, normalised gradient chain, backward pair
    kernel, a repartition after every 2 epochs, 3 epochs = 24 phases.  Device-side copies
    captured into the graph after every phase (Trainer.phase_probe) record theta, the aggregated
    update and the hidden activations; every phase's update is compared with the oracle's at the
    GPU's own theta (step-local, as test_epoch_parity) with the kernels' ReLU decisions, each
    checked against the R16b bf16 flip bound."""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000)     # depth 8
    assert wl.depth == 8
    ds = gen.make_dataset(wl)
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    lr, rep, epochs = 0.05, 2, 3
    P = wl.chunks
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr="uniform", lr=lr, repartition_every=rep, dtype="bf16")
    tr.graph_eager_min_nnz = 0 if eager_capture else 1 << 62
    nmax = ds.wl.n
    snap_theta = [torch.empty_like(tr.theta) for _ in range(P)]
    snap_grad = [torch.empty_like(tr.grad) for _ in range(P)]
    snap_h = [[torch.zeros(nmax, wl.dims_pad[l], dtype=torch.bfloat16, device="cuda") for l in range(wl.depth)]
              for _ in range(P)]

    def probe(i, w):
        n = tr.parts[w].n_core
        snap_theta[i].copy_(tr.theta)
        snap_grad[i].copy_(tr.grad)
        for l in range(1, wl.depth):
            snap_h[i][l][:n].copy_(tr.H[l][:n])

    tr.phase_probe = probe
    thetas, ghat, masks, sizes = [_logical(tr, tr.theta)], [], [], []
    for e in range(epochs):
        tr.run_epoch_graph()
        torch.cuda.synchronize()
        for i in range(P):
            n = tr.parts[i].n_core
            ghat.append(_logical(tr, snap_grad[i]))
            thetas.append(_logical(tr, snap_theta[i]))
            masks.append([(snap_h[i][l][:n, :wl.dims[l]].float() > 0).cpu().numpy().astype(np.float64)
                          for l in range(1, wl.depth)])
    tr.check()
    assert tr.graph is not None and tr.graph_launches > 0
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    sched = Po.sweep_schedule(P, P)
    X = torch.from_numpy(ds.x[:, :wl.F]).to(torch.bfloat16).double().numpy()
    shapes = [[w.shape for w in ws] for ws in _oracle_weights(ds, wl.dims)]
    flips = 0
    for k in range(epochs * P):
        e, w = divmod(k, P)
        b, s = sched[(e // rep) % len(sched)][w]
        part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
        _, g, _, cache = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                                Mo.unflatten(thetas[k], shapes), masks[k])
        flips += assert_flips_bounded(cache, "bf16", f"phase {k}")
        ref = Co.aggregate([Tr.partition_factor("uniform", part)], [g], 1)
        assert err(ghat[k], ref) <= TOL["bf16"], (k, err(ghat[k], ref))
        # the SGD step the graph applied is lr times that update
        assert err(thetas[k] - thetas[k + 1], lr * ghat[k]) <= 1e-2, k
    print(f"{epochs * P} graph-replayed phases vs the oracle, {flips} ReLU decisions within the R16b bound")


@pytest.mark.parametrize("width", [128, 112, 80, 96])
@pytest.mark.parametrize("mode", ["plain", "node", "halo"])
def test_spmm_tma_bitwise_equals_row_group(G, ctx, prod, width, mode):
    """The TMA-gather SpMM (spmm_tma.cu, ctx variant "spmm" = 4, for bf16 unweighted aggregations
    of 80..128 wide rows) sums every row's neighbours in the same edge order as the row-group
    kernel and applies the same epilogue, so forward h_out (self term, row scale, node-level
    neighbour scale, ReLU) and the backward dz_in / dW agree BIT FOR BIT with the row-group
    kernel (the default, variant 0) -- on induced-core partitions (hub rows split into 256-edge segments)
    and on halo-1 partitions (forward on A, backward on the stored transpose)."""
    rp, col, x, y, tr = upload(prod)
    ch = torch.empty(prod.wl.n, dtype=torch.int32, device="cuda")
    G.grappa_partition(ctx, prod.wl.n, 8, gen.seed_of("chunks"), ch)
    part = G.grappa_repartition(ctx, rp, col, x.to(torch.bfloat16), "bf16", ch, 8, 2, 5, tr, y,
                                halo=(mode == "halo"))
    assert part.info.n_heavy > 0 or mode == "halo"
    n, f_in = part.n_core, 64
    g = torch.Generator(device="cuda").manual_seed(width)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(torch.bfloat16)
    w = (torch.randn(f_in, width, device="cuda", generator=g) / 8).contiguous()
    dz = (torch.randn(n, width, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    flags = G.LAYER_NODE_LEVEL if mode == "node" else 0
    outs = []
    for variant in (4, 0):
        ctx.set_variant("spmm", variant)
        ws = torch.empty(G.layer_ws_bytes(part, "gcn", f_in, width, "bf16"), dtype=torch.uint8, device="cuda")
        h_out = torch.empty(n, width, device="cuda", dtype=torch.bfloat16)
        G.grappa_layer_fwd_ex(ctx, part, "gcn", f_in, width, True, h_in, w, h_out, None, ws, "bf16", flags)
        dw = torch.empty_like(w)
        dz_in = torch.empty(n, f_in, device="cuda", dtype=torch.bfloat16)
        G.grappa_layer_bwd_ex(ctx, part, "gcn", f_in, width, True, dz, h_in, w, None, dw, dz_in, ws, "bf16",
                              flags | G.BWD_DZ_OUT_NORMED | G.BWD_DZ_IN_NORMED if mode != "node" else flags)
        torch.cuda.synchronize()
        outs.append((h_out.view(torch.int16).clone(), dz_in.view(torch.int16).clone(), dw.clone()))
    ctx.set_variant("spmm", 0)
    (a_h, a_dz, a_dw), (b_h, b_dz, b_dw) = outs
    assert torch.equal(a_h, b_h)
    assert torch.equal(a_dz, b_dz)
    assert torch.equal(a_dw, b_dw)


@pytest.mark.parametrize("C,dtype", [(8, "bf16"), (4, "f32"), (2, "bf16"), (80, "bf16")])
def test_repartition_batch_bitexact(G, ctx, prod, C, dtype):
    """grappa_repartition_batch (all partitions of a switch, two host syncs; with the run's
    grappa_index or a temporary one) builds every partition bit for bit as grappa_repartition and
    the oracle do; the index's per-chunk counts and degree sums are exact -- CSR, maps, degrees, norms, node weights,
    seeds, labels, gathered features, split-row plan sizes, coverage statistics -- reusing the
    previous switch's partition objects; chunk sizes that disagree with the map are rejected."""
    rp, col, x, y, tr = upload(prod)
    seed = gen.seed_of("chunks")
    ch = torch.empty(prod.wl.n, dtype=torch.int32, device="cuda")
    sizes = G.grappa_partition(ctx, prod.wl.n, C, seed, ch)
    chunk_of = Po.make_chunks(prod.wl.n, C, seed)
    xt = x.to(torch.bfloat16) if dtype == "bf16" else x
    sched = Po.sweep_schedule(C, C)
    parts = None
    index = G.Index(ctx, rp, col, ch, C)        # the engine's path: one index for the whole run
    assert index.query()[0] == list(sizes)
    deg = np.diff(prod.rowptr)
    assert index.query()[1] == [int(deg[chunk_of == c].sum()) for c in range(C)]
    for t in range(min(3, len(sched))):
        pairs = sched[t][:8]
        parts = G.grappa_repartition_batch(ctx, rp, col, xt, dtype, ch, C, pairs, tr, y, parts, chunk_sizes=sizes,
                                           index=index if t != 1 else None)
        for (b, s), p in zip(pairs, parts):
            one = G.grappa_repartition(ctx, rp, col, xt, dtype, ch, C, b, s, tr, y)
            ref = Po.induced_partition(prod.rowptr, prod.col, chunk_of, b, s, prod.train)
            assert np.array_equal(p.rowptr.cpu().numpy(), ref["rowptr"])
            assert np.array_equal(p.col.cpu().numpy(), ref["col"])
            assert np.array_equal(p.seeds.cpu().numpy(), ref["seeds"])
            for name in ("rowptr", "col", "core_global", "d_l", "d_g", "norm_gcn", "norm_sage", "seeds", "labels",
                         "node_w"):
                assert torch.equal(getattr(p, name), getattr(one, name)), name
            assert torch.equal(p.x.view(torch.int16) if dtype == "bf16" else p.x,
                               one.x.view(torch.int16) if dtype == "bf16" else one.x)
            for f in ("n_core", "nnz", "n_seeds", "n_heavy", "n_slots", "D", "c_uniform", "c_resampling",
                      "c_resampling_hm"):
                assert getattr(p.info, f) == getattr(one.info, f), f
    with pytest.raises(G.GrappaError, match="E_ARG"):       # an index of another graph
        G.grappa_repartition_batch(ctx, rp, col.clone(), xt, dtype, ch, C, sched[0][:8], tr, y, chunk_sizes=sizes,
                                   index=index)
    bad = list(sizes)
    bad[sched[0][0][0]] += 1
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_repartition_batch(ctx, rp, col, xt, dtype, ch, C, sched[0][:8], tr, y, chunk_sizes=bad)
    with pytest.raises(G.GrappaError, match="E_EMPTY"):
        G.grappa_repartition_batch(ctx, rp, col, xt, dtype, ch, C, sched[0][:8], torch.zeros_like(tr), y,
                                   chunk_sizes=sizes)


def test_controller_drives_switches(G, ctx, prod):
    """§3.5 controller in the training loop (R32): the trainer feeds every phase's coverage
    (c_uniform of its partition) to the controller and switches super-epochs when it says so; the
    switch epochs equal those of the oracle controller fed the oracle partitions' coverages."""
    from oracle.controller import Controller as OC
    from paper_2602_01872_b200.controller import Controller
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    # a deficit threshold between the partitions' coverages makes some partitions fire early
    P = wl.chunks
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    sched = Po.sweep_schedule(P, P)
    cov = {}
    for t in range(len(sched)):
        for w, (b, s) in enumerate(sched[t]):
            part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
            cov[(t, w)] = Co.c_uniform(part["d_l"][part["seeds"]], part["d_g"][part["seeds"]])
    vals = sorted(cov.values())
    m = len(vals) // 2
    thr = 1.0 - 0.5 * (vals[m - 1] + vals[m])       # between two coverages: no ties at 1e-12
    mk = lambda: Controller(epochs_total=40, num_chunks=P, deficit_threshold=thr, streak_threshold=2)
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, P, gen.seed_of("chunks"),
                 corr="uniform", lr=0.0, controller=mk())
    got = []
    for _ in range(6):
        tr.run_epoch()
        got.append(tr.t)
    oc = OC(40, P, deficit_threshold=thr, streak_threshold=2)
    t, ref = 1, []
    for _ in range(6):
        ref.append(t)
        for w in range(P):
            oc.observe(w, cov[((t - 1) % len(sched), w)])
        if oc.end_epoch():
            t += 1
    assert got == ref and len(set(ref)) > 1, (got, ref)
