"""Full-size parity (BASELINE.json configs[2], the metric's config) in the launch configuration
bench.py times (bf16 storage, default kernel variants, the engine's Trainer): the ogbn-products
shaped graph (2,449,029 nodes, 123.7M directed edges), GCN-8, P = 8.

* chunking and the first super-epoch partition of worker 0 bit-exact against the oracle over
  every node and edge (2.45M chunk ids, 612k core rows, 7.7M local edges, degrees, seeds);
* one Alg. 1 phase end to end: the aggregated update of partition 0 through all 8 layers vs the
  oracle's f64 gradient on the same partition, with the ReLU decisions the kernels took (R16b),
  at the bf16 bar 2e-2;
* one layer of the same partition checked on 10^4 sampled rows computed one by one from the
  GPU's own inputs (forward), and dW reduced over all 612k rows in f64 (backward).
Slow (~1-2 min: generation + a full f64 oracle pass); marked gpu."""
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


def err(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30))


@pytest.fixture(scope="module")
def setup():
    import paper_2602_01872_b200 as G
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    G.load()
    wl = gen.WORKLOADS["products"]
    ds = gen.make_dataset(wl)
    ctx = G.Context(0)
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr=wl.correction, lr=0.003,
                 repartition_every=wl.repartition_every, dtype="bf16")
    tr.repartition(1)
    torch.cuda.synchronize()
    yield G, wl, ds, ctx, tr
    ctx.close()


def test_fullsize_partition_bitexact(setup):
    G, wl, ds, ctx, tr = setup
    chunk_of = Po.make_chunks(wl.n, wl.chunks, gen.seed_of("chunks"))
    assert np.array_equal(tr.chunk_of.cpu().numpy(), chunk_of)
    b, s = Po.sweep_schedule(wl.chunks, wl.chunks)[0][0]
    ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
    p = tr.parts[0]
    assert p.n_core == ref["core"].size and p.nnz == ref["col"].size
    assert np.array_equal(p.core_global.cpu().numpy(), ref["core"])
    assert np.array_equal(p.rowptr.cpu().numpy(), ref["rowptr"])
    assert np.array_equal(p.col.cpu().numpy(), ref["col"])
    assert np.array_equal(p.d_l.cpu().numpy(), ref["d_l"])
    assert np.array_equal(p.d_g.cpu().numpy(), ref["d_g"])
    assert np.array_equal(p.seeds.cpu().numpy(), ref["seeds"])
    s_dl, s_dg = ref["d_l"][ref["seeds"]], ref["d_g"][ref["seeds"]]
    assert p.info.D == int(np.sum((s_dg - s_dl)[s_dl > 0]))
    assert p.info.c_resampling == Co.c_resampling(s_dl, s_dg)
    # bf16 features gathered bit for bit
    xb = torch.from_numpy(ds.x).to(torch.bfloat16)
    idx = torch.from_numpy(ref["core"])
    assert torch.equal(p.x.cpu().view(torch.int16), xb[idx].view(torch.int16))


def test_fullsize_layer_sampled_rows(setup):
    """layer 2 of GCN-8 (128 -> 128) on the full partition: forward checked on 10^4 sampled rows
    recomputed one by one in f64 from the GPU's own input; dW over all rows in f64."""
    G, wl, ds, ctx, tr = setup
    p = tr.parts[0]
    n = p.n_core
    g = torch.Generator(device="cuda").manual_seed(11)
    h_in = torch.randn(n, 128, device="cuda", generator=g).relu().to(torch.bfloat16)
    w = (torch.randn(128, 128, device="cuda", generator=g) / math.sqrt(128)).contiguous()
    h_out = torch.empty(n, 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(G.layer_ws_bytes(p, "gcn", 128, 128, "bf16"), dtype=torch.uint8, device="cuda")
    G.grappa_layer_fwd(ctx, p, "gcn", 128, 128, True, h_in, w, h_out, None, ws, "bf16")
    dz = (torch.randn(n, 128, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    dw = torch.empty_like(w)
    dz_in = torch.empty(n, 128, device="cuda", dtype=torch.bfloat16)
    G.grappa_layer_bwd(ctx, p, "gcn", 128, 128, True, dz, h_in, w, None, dw, dz_in, ws, "bf16")
    torch.cuda.synchronize()
    rp, col = p.rowptr.cpu().numpy(), p.col.cpu().numpy()
    nrm = 1.0 / np.sqrt(np.diff(rp) + 1.0)
    H = h_in.float().cpu().numpy().astype(np.float64)
    W = w.cpu().numpy().astype(np.float64)
    out = h_out.float().cpu().numpy()
    rows = np.random.default_rng(5).choice(n, 10_000, replace=False)
    T = None
    ref = np.empty((rows.size, 128))
    for k, v in enumerate(rows):                           # Z_v = n_v (n_v h_v + sum n_u h_u) W
        nb = col[rp[v]:rp[v + 1]]
        a = nrm[v] * (nrm[v] * H[v] + (nrm[nb, None] * H[nb]).sum(axis=0))
        ref[k] = np.maximum(a @ W, 0.0)
    assert err(out[rows], ref) <= 2e-2
    # dW = h_in^T (Ahat dz) over every row, f64
    op = Mo.gcn_operator(rp, col, n)
    dT = op.T @ dz.float().cpu().numpy().astype(np.float64)
    assert err(dw.cpu().numpy(), H.T @ dT) <= 2e-2
    del T


def test_fullsize_phase_update(setup):
    """one Alg. 1 phase of the bench's configuration (partition 0, all 8 layers, loss,
    backward, resampling factor): aggregated update vs the oracle in f64."""
    G, wl, ds, ctx, tr = setup
    theta0 = tr.theta.clone()
    tr.phase_step(0, 0, 1)
    torch.cuda.synchronize()
    ctx.check()
    p = tr.parts[0]
    n = p.n_core
    sp = tr.spec
    masks = [(tr.H[l][:n, :wl.dims[l]] > 0).cpu().numpy() for l in range(1, wl.depth)]
    mats, off = [], 0
    for l, (a, b) in enumerate(sp.layer_shapes()):
        blk = tr.grad[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
        off += a * b
        mats.append([blk[:wl.dims[l], :wl.dims[l + 1]]])
    ghat = Mo.flatten(mats)
    chunk_of = tr.chunk_of.cpu().numpy()
    b, s = Po.sweep_schedule(wl.chunks, wl.chunks)[0][0]
    part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
    X = torch.from_numpy(ds.x[:, :wl.F]).to(torch.bfloat16).double().numpy()[part["core"]]
    W0 = [[np.asarray(w, np.float64)[:wl.dims[l], :wl.dims[l + 1]] for w in ws]
          for l, ws in enumerate(ds.weights)]
    _, g, _, cache = Mo.partition_loss_grad(wl.arch, part, X, ds.y[part["core"]], W0, masks)
    assert_flips_bounded(cache, "bf16", "fullsize phase")
    ref = Co.aggregate([Tr.partition_factor(wl.correction, part)], [g], 1)
    assert err(ghat, ref) <= 2e-2
    tr.theta.copy_(theta0)
