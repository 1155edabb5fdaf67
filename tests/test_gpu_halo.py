"""GPU parity of halo-1 partitions (readings
R33/R34) through the C ABI vs the f64 oracle: bit-exact partition (local ids, CSR, degrees,
seeds, gathered features) and transpose; 1e-4 / 2e-2 on layers (forward on A_loc, backward on
its transpose) and on Alg. 1's aggregated updates."""
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
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3)
    return gen.make_dataset(wl)


def _part(G, ctx, ds, C, b, s, dtype="f32", part=None):
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    x = torch.from_numpy(ds.x).to(d)
    x = x.to(torch.bfloat16) if dtype == "bf16" else x
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    return G.grappa_repartition(ctx, rp, col, x, dtype, ch, C, b, s, torch.from_numpy(ds.train).to(d),
                                torch.from_numpy(ds.y).to(d), part, halo=True)


@pytest.mark.parametrize("C,pairs", [(8, [(0, 1), (3, 7), (6, 2)]), (2, [(0, 1)]), (4, [(1, 3)])])
def test_halo_repartition_bitexact(G, ctx, prod, C, pairs):
    ds = prod
    chunk_of = Po.make_chunks(ds.wl.n, C, gen.seed_of("chunks"))
    part = None
    for b, s in pairs:
        part = _part(G, ctx, ds, C, b, s, part=part)
        ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train, halo=True)
        n = ref["core"].size
        assert part.n_core == n and part.n_halo == n - ref["n_core"]
        assert np.array_equal(part.core_global.cpu().numpy(), ref["core"])
        assert np.array_equal(part.rowptr.cpu().numpy(), ref["rowptr"])
        assert np.array_equal(part.col.cpu().numpy(), ref["col"])
        assert np.array_equal(part.d_l.cpu().numpy(), ref["d_l"])
        assert np.array_equal(part.d_g.cpu().numpy(), ref["d_g"])
        assert np.array_equal(part.seeds.cpu().numpy(), ref["seeds"])
        assert np.array_equal(part.labels.cpu().numpy(), ds.y[ref["core"]])
        assert np.array_equal(part.x.cpu().numpy(), ds.x[ref["core"]])
        assert np.array_equal(part.norm_gcn.cpu().numpy(), (1.0 / np.sqrt(ref["d_l"] + 1.0)).astype(np.float32))
        # every seed is a core node with its full neighbourhood: all batch factors are 1 (R33)
        assert part.info.D == 0 and part.info.c_uniform == 1.0 and part.info.c_resampling == 1.0
        if C == 2:
            assert part.n_halo == 0
        # the transpose: sources of every column, ascending local id
        rows = np.repeat(np.arange(n), np.diff(ref["rowptr"]))
        o = np.lexsort((rows, ref["col"]))
        t_rp = np.searchsorted(ref["col"][o], np.arange(n + 1))
        assert np.array_equal(part.t_rowptr.cpu().numpy(), t_rp)
        assert np.array_equal(part.t_col.cpu().numpy(), rows[o])


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("f_in,f_out", [(112, 128), (128, 48)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("flags", ["plain", "normed", "node"])
def test_halo_layer_parity(G, ctx, prod, arch, f_in, f_out, dtype, flags):
    if flags == "normed" and arch == "sage":
        pytest.skip("normalised gradients are GCN-only")
    part = _part(G, ctx, prod, 8, 2, 5, dtype)
    n = part.n_core
    assert part.n_halo > 0
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(f_in * 7 + f_out)
    h_in = torch.randn(n, f_in, device="cuda", generator=g).relu().to(tdt)
    m = 1 if arch == "gcn" else 2
    w = (torch.randn(m * f_in, f_out, device="cuda", generator=g) / math.sqrt(f_in)).contiguous()
    h_out = torch.empty(n, f_out, device="cuda", dtype=tdt)
    saved = torch.empty(max(1, G.layer_saved_bytes(part, arch, f_in, f_out, dtype)), dtype=torch.uint8,
                        device="cuda")
    ws = torch.empty(G.layer_ws_bytes(part, arch, f_in, f_out, dtype), dtype=torch.uint8, device="cuda")
    fl = G.LAYER_NODE_LEVEL if flags == "node" else 0
    G.grappa_layer_fwd_ex(ctx, part, arch, f_in, f_out, True, h_in, w, h_out, saved, ws, dtype, fl)
    nrm = part.norm_gcn.double().cpu().numpy()
    dz = torch.randn(n, f_out, device="cuda", generator=g) * 1e-3
    normed = flags == "normed"
    dz_k = (dz * part.norm_gcn[:, None]).to(tdt) if normed else dz.to(tdt)
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, f_in, device="cuda", dtype=tdt)
    bfl = fl | ((G.BWD_DZ_OUT_NORMED | G.BWD_DZ_IN_NORMED) if normed else 0)
    G.grappa_layer_bwd_ex(ctx, part, arch, f_in, f_out, True, dz_k, h_in, w, saved, dw, dz_in, ws, dtype, bfl)
    torch.cuda.synchronize()
    rp, cl = part.rowptr.cpu().numpy(), part.col.cpu().numpy()
    node_w = Co.node_weights(part.d_l.cpu().numpy(), part.d_g.cpu().numpy()) if flags == "node" else None
    op = Mo.operator(arch, rp, cl, n, node_w)
    H, W = _np(h_in), _np(w)
    Ws = [W] if arch == "gcn" else [W[:f_in], W[f_in:]]
    P, Z, Hn = Mo.layer_forward(arch, op, H, Ws, True)
    tol = TOL[dtype]
    assert err(_np(h_out), Hn) <= tol
    dz_ref = _np(dz_k) / nrm[:, None] if normed else _np(dz_k)
    grads, dH = Mo.layer_backward(arch, op, H, P, Ws, dz_ref)      # uses op.T (non-symmetric)
    assert err(_np(dw), np.concatenate(grads, axis=0)) <= tol
    ref_in = dH * (H > 0)
    if normed:
        ref_in = nrm[:, None] * ref_in
    assert err(_np(dz_in), ref_in) <= tol
    # the transpose matters: the symmetric-operator backward would be off
    _, dH_sym = Mo.layer_backward(arch, op.T.tocsr(), H, P, Ws, dz_ref)
    assert err(dH_sym * (H > 0) * (nrm[:, None] if normed else 1.0), ref_in) > 10 * tol


def test_halo_epoch_parity(G, ctx, prod):
    """Alg. 1 with halo-1 partitions, P = 8, M = 1, one epoch (fp32): every phase's aggregated
    update vs the oracle's gradient on its halo-1 partition at the GPU's own theta (R16b)."""
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ds = prod
    wl = ds.wl
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    lr = 0.05
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr="resampling", lr=lr, repartition_every=1, halo=True)

    def logical(flat):
        mats, off = [], 0
        for l, (a, b) in enumerate(spec.layer_shapes()):
            blk = flat[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
            off += a * b
            mats.append([blk[:wl.dims[l], :wl.dims[l + 1]]])
        return Mo.flatten(mats)

    thetas, ghat, masks = [logical(tr.theta)], [], []

    def grab():
        ghat.append(logical(tr.grad))
        thetas.append(logical(tr.theta))
        n = tr.parts[len(masks)].n_core
        masks.append([(tr.H[l][:n, :wl.dims[l]] > 0).cpu().numpy().astype(np.float64)
                      for l in range(1, wl.depth)])

    tr.run_epoch(on_phase=grab)
    torch.cuda.synchronize()
    ctx.check()
    P = wl.chunks
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    sched = Po.sweep_schedule(P, P)
    X = ds.x[:, :wl.F].astype(np.float64)
    Wref = [[np.asarray(w, np.float64)[:wl.dims[l], :wl.dims[l + 1]] for w in ws]
            for l, ws in enumerate(ds.weights)]
    shapes = [[w.shape for w in ws] for ws in Wref]
    for k in range(P):
        b, s = sched[0][k]
        part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train, halo=True)
        _, g, _, cache = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                                Mo.unflatten(thetas[k], shapes), masks[k])
        assert_flips_bounded(cache, "f32", f"halo phase {k}")
        c = Tr.partition_factor("resampling", part)
        assert c == 1.0
        assert err(ghat[k], Co.aggregate([c], [g], 1)) <= 1e-4, k
        assert err(thetas[k] - thetas[k + 1], lr * ghat[k]) <= 1e-3
