"""GPU parity of GAT layers (reading R35) through the C ABI vs the f64
oracle: layer-local forward / backward (dW including the attention vectors, dh) on induced-core
and halo-1 partitions, fp32 (1e-4) and bf16 (2e-2), and Alg. 1 epochs."""
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
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3, arch="gat")
    return gen.make_dataset(wl)


def _part(G, ctx, ds, C, b, s, dtype="f32", halo=False):
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    x = torch.from_numpy(ds.x).to(d)
    x = x.to(torch.bfloat16) if dtype == "bf16" else x
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    return G.grappa_repartition(ctx, rp, col, x, dtype, ch, C, b, s, torch.from_numpy(ds.train).to(d),
                                torch.from_numpy(ds.y).to(d), halo=halo)


@pytest.mark.parametrize("f_in,f_out", [(112, 128), (128, 48), (128, 128)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("halo", [False, True])
def test_gat_layer_parity(G, ctx, prod, f_in, f_out, dtype, halo):
    part = _part(G, ctx, prod, 8, 2, 5, dtype, halo)
    n = part.n_core
    assert part.info.n_heavy > 0                     # hub rows take the block-per-row kernels
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in * 3 + f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    w = torch.randn(f_in + 2, f_out, device="cuda", generator=g)
    w[:f_in] /= math.sqrt(f_in)
    w[f_in:] *= 0.3
    w = w.contiguous()
    h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
    saved = torch.empty(G.layer_saved_bytes(part, "gat", f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, "gat", f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    G.grappa_layer_fwd_ex(ctx, part, "gat", f_in, f_out, True, h_in, w, h_out, saved, ws, dtype, 0)
    dz = (torch.randn(n, f_out, device="cuda", generator=g) * 1e-3).to(tdt)
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
    G.grappa_layer_bwd_ex(ctx, part, "gat", f_in, f_out, True, dz, h_in, w, saved, dw, dz_in, ws, dtype, 0)
    torch.cuda.synchronize()
    op = Mo.operator("gat", part.rowptr.cpu().numpy(), part.col.cpu().numpy(), n)
    H, W = _np(h_in), _np(w)
    Ws = [W[:f_in], W[f_in:]]
    P, Z, Hn = Mo.layer_forward("gat", op, H, Ws, True)
    tol = TOL[dtype]
    assert err(_np(h_out), Hn) <= tol
    grads, dH = Mo.layer_backward("gat", op, H, P, Ws, _np(dz))
    ref_dw = np.concatenate(grads, axis=0)
    assert err(_np(dw)[:f_in], ref_dw[:f_in]) <= tol
    assert err(_np(dw)[f_in:], ref_dw[f_in:]) <= tol          # attention vectors
    assert err(_np(dz_in), dH * (H > 0)) <= tol


def test_gat_flags(G, ctx, prod):
    part = _part(G, ctx, prod, 8, 2, 5)
    n = part.n_core
    h = torch.zeros(n, 16, device="cuda")
    w = torch.zeros(18, 16, device="cuda")
    saved = torch.empty(G.layer_saved_bytes(part, "gat", 16, 16, "f32"), dtype=torch.uint8, device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, "gat", 16, 16, "f32"), dtype=torch.uint8, device="cuda")
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_layer_fwd_ex(ctx, part, "gat", 16, 16, True, h, w, h.clone(), saved, ws, "f32",
                              G.LAYER_NODE_LEVEL)
    with pytest.raises(G.GrappaError, match="E_SHAPE"):
        big = torch.empty(G.layer_ws_bytes(part, "gat", 16, 256, "f32"), dtype=torch.uint8, device="cuda")
        sv = torch.empty(G.layer_saved_bytes(part, "gat", 16, 256, "f32"), dtype=torch.uint8, device="cuda")
        G.grappa_layer_fwd_ex(ctx, part, "gat", 16, 256, True, h, torch.zeros(18, 256, device="cuda"),
                              torch.empty(n, 256, device="cuda"), sv, big, "f32", 0)


@pytest.mark.parametrize("dtype,halo", [("f32", False), ("f32", True), ("bf16", False)])
def test_gat_epoch_parity(G, ctx, prod, dtype, halo):
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=1, dtype=dtype, halo=halo)

    def logical(flat):
        mats, off = [], 0
        for l, (a, b) in enumerate(spec.layer_shapes()):
            blk = flat[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
            off += a * b
            fi, fo, fip = wl.dims[l], wl.dims[l + 1], wl.dims_pad[l]
            mats.append([blk[:fi, :fo], blk[fip:fip + 2, :fo]])
        return Mo.flatten(mats)

    thetas, ghat, masks = [logical(tr.theta)], [], []

    def grab():
        ghat.append(logical(tr.grad))
        thetas.append(logical(tr.theta))
        n = tr.parts[len(masks)].n_core
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
    W0 = [[np.asarray(ws[0], np.float64)[:wl.dims[l], :wl.dims[l + 1]],
           np.asarray(ws[1], np.float64)[:2, :wl.dims[l + 1]]] for l, ws in enumerate(ds.weights)]
    shapes = [[w.shape for w in ws] for ws in W0]
    for k in range(P):
        b, s = sched[0][k]
        part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train, halo=halo)
        _, g, _, cache = Mo.partition_loss_grad("gat", part, X[part["core"]], ds.y[part["core"]],
                                                Mo.unflatten(thetas[k], shapes), masks[k])
        assert_flips_bounded(cache, dtype, f"gat phase {k}")
        ref = Co.aggregate([Tr.partition_factor("uniform", part)], [g], 1)
        assert err(ghat[k], ref) <= TOL[dtype], k
