"""Degenerate inputs through the C ABI vs the oracle: an edgeless graph (every partition has
nnz = 0, every seed d_l = d_g = 0 -> c = 1), a star (one hub of degree 6000: split SpMM rows on
both the forward and the backward, hub picks in the sampler), and single-seed partitions."""
import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import sampler as Sa
from oracle import train as Tr

pytestmark = pytest.mark.gpu


def err(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30))


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


def _dataset(rowptr, col, n, arch, seed=0, train_every=3):
    wl = gen.small_workload("products", n=n, scale=max(4, (n - 1).bit_length()), num_samples=10,
                            arch=arch, depth=2, hidden=32, chunks=4)
    rng = np.random.default_rng(seed)
    x = np.zeros((n, wl.dims_pad[0]), np.float32)
    x[:, :wl.F] = rng.uniform(-1, 1, (n, wl.F)).astype(np.float32)
    y = rng.integers(0, wl.K, n).astype(np.int32)
    train = (np.arange(n) % train_every == 0).astype(np.uint8)
    return wl, gen.Dataset(wl, rowptr, col, x, y, train, gen.init_weights(wl, 7))


def _epoch_parity(G, wl, ds, corr):
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    ctx = G.Context(0)
    spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
    lr = 0.05
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr=corr, lr=lr, repartition_every=1)
    thetas = []

    def logical():
        mats, off = [], 0
        for l, (a, b) in enumerate(spec.layer_shapes()):
            blk = tr.theta[off:off + a * b].view(a, b).cpu().numpy().astype(np.float64)
            off += a * b
            fi, fo, fip = wl.dims[l], wl.dims[l + 1], wl.dims_pad[l]
            if wl.arch == "gcn":
                mats.append([blk[:fi, :fo]])
            elif wl.arch == "gat":
                mats.append([blk[:fi, :fo], blk[fip:fip + 2, :fo]])
            else:
                mats.append([blk[:fi, :fo], blk[fip:fip + fi, :fo]])
        return Mo.flatten(mats)

    thetas.append(logical())
    tr.run_epoch(on_phase=lambda: thetas.append(logical()))
    torch.cuda.synchronize()
    ctx.check()
    chunk_of = Po.make_chunks(wl.n, wl.chunks, gen.seed_of("chunks"))
    W0 = [[np.asarray(w, np.float64)[:wl.dims[l], :wl.dims[l + 1]] for w in ws]
          for l, ws in enumerate(ds.weights)]
    final, recs = Tr.run(wl.arch, ds.rowptr, ds.col, ds.x[:, :wl.F].astype(np.float64), ds.y, ds.train,
                         W0, chunk_of, wl.chunks, wl.chunks, 1, corr, lr, 1, 1)
    assert err(thetas[-1], Mo.flatten(final)) <= 1e-4
    ctx.close()
    return recs


@pytest.mark.parametrize("arch", ["gcn", "sage", "gat"])
def test_edgeless_graph(G, arch):
    n = 400
    rowptr = np.zeros(n + 1, np.int64)
    col = np.zeros(0, np.int32)
    wl, ds = _dataset(rowptr, col, n, arch)
    recs = _epoch_parity(G, wl, ds, "resampling")
    assert all(c == 1.0 for r in recs for c in r["c"])          # D = 0 -> guard -> 1


@pytest.mark.parametrize("arch", ["gcn", "sage", "gat"])
def test_star_hub(G, arch):
    n = 6001                                                  # node 0 linked to every other node
    wl, ds = _dataset(*gen.csr_from_edges(n, [(0, v) for v in range(1, n)]), n, arch)
    _epoch_parity(G, wl, ds, "uniform")


def test_star_sampler_and_single_seed(G):
    n = 6001
    rowptr, col = gen.csr_from_edges(n, [(0, v) for v in range(1, n)])
    wl, ds = _dataset(rowptr, col, n, "sage", train_every=n + 1)   # one train node: node 0
    ctx = G.Context(0)
    d = "cuda"
    ch = torch.empty(n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, n, 2, gen.seed_of("chunks"), ch)
    chunk_of = Po.make_chunks(n, 2, gen.seed_of("chunks"))
    ref = Po.induced_partition(rowptr, col, chunk_of, 0, 1, ds.train)
    assert ref["seeds"].tolist() == [0]
    p = G.grappa_repartition(ctx, torch.from_numpy(rowptr).to(d), torch.from_numpy(col).to(d),
                             torch.from_numpy(ds.x).to(d), "f32", ch, 2, 0, 1, torch.from_numpy(ds.train).to(d),
                             torch.from_numpy(ds.y).to(d))
    assert p.n_seeds == 1
    for fan in ([5, 3], [16, 16]):
        b = G.grappa_sample(ctx, p, torch.tensor([0], dtype=torch.int32, device=d), fan, 3, 0, 0)
        blocks = Sa.sample_batch(ref, np.array([0]), fan, 3, 0, 0)
        for gb, ob in zip(b.blocks, blocks):
            assert np.array_equal(gb["src"].cpu().numpy(), ob["src"])
            assert np.array_equal(gb["col"].cpu().numpy(), ob["col"])
        d_l, d_g, s = Sa.batch_stats(ref, blocks)
        assert b.factors["resampling"] == Co.c_resampling(d_l, d_g, s)
    ctx.close()
