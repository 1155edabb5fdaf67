"""Pins for oracle step a10 (isolated mini-batch sampling + SAGE on blocks) -- CPU only.

Pins: SPEC hand cases (fanout >= degree returns every neighbour, isolated target returns
none, the triangle draw S:204), the epoch iterator contract, conditional uniformity
of the draw (each local neighbour sampled with frequency f/d within 4 sigma), the
reduction of a one-batch, full-fanout mini-batch to the full-graph SAGE layer of
oracle.model (itself pinned against a dense re-derivation), and finite differences.
"""
import numpy as np
import pytest

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import sampler as Sa


def whole(n, edges, train=None):
    rp, col = gen.csr_from_edges(n, edges)
    ch = np.arange(n) % 2
    return Po.induced_partition(rp, col, ch.astype(np.int32), 0, 1,
                                np.ones(n, np.uint8) if train is None else train)


def test_triangle_and_degenerate_cases():
    p = whole(3, [(0, 1), (1, 2), (0, 2)])
    blocks = Sa.sample_batch(p, [0], [2], 7, 0, 0)
    assert blocks[0]["src"].tolist() == [0, 1, 2] and blocks[0]["col"].tolist() == [1, 2]
    p = whole(4, [(0, 1), (0, 2), (0, 3)])
    b = Sa.sample_batch(p, [0], [5], 7, 0, 0)[0]                        # S:202 d <= f
    assert sorted(b["src"][b["col"]].tolist()) == [1, 2, 3]
    p = whole(3, [(1, 2)])
    b = Sa.sample_batch(p, [0], [3], 7, 0, 0)[0]                        # S:203 d_l = 0
    assert b["rowptr"].tolist() == [0, 0] and b["src"].tolist() == [0]


def test_structure_and_prefix_order():
    rp, col = gen.rmat(10, 1000, 12000, 5, 6)
    ch = Po.make_chunks(1000, 4, 3)
    p = Po.induced_partition(rp, col, ch, 0, 2, (np.arange(1000) % 3 == 0).astype(np.uint8))
    batches = Sa.epoch_batches(p, 11, 0, 50)
    blocks = Sa.sample_batch(p, batches[0], [6, 4, 3], 11, 0, 0)
    fan = [6, 4, 3]
    for l, b in enumerate(blocks):
        assert np.array_equal(b["src"][:b["n_dst"]], b["dst"])           # targets are a prefix
        assert np.all(np.diff(b["src"][b["n_dst"]:]) > 0)                  # new ones ascending
        for i, v in enumerate(b["dst"]):
            pos = b["col"][b["rowptr"][i]:b["rowptr"][i + 1]]
            assert np.all(np.diff(pos) > 0)                                 # distinct, ordered
            nb = set(p["col"][p["rowptr"][v]:p["rowptr"][v + 1]].tolist())
            assert set(b["src"][pos].tolist()) <= nb                        # local neighbours only
            assert len(pos) == min(fan[l], len(nb))
        if l + 1 < len(blocks):
            assert np.array_equal(blocks[l + 1]["src"], b["dst"])


def test_epoch_iterator_contract():
    p = whole(23, [(i, i + 1) for i in range(22)])
    b1 = Sa.epoch_batches(p, 5, 0, 4)
    assert [len(x) for x in b1] == [4, 4, 4, 4, 4, 3]                      # S:220 arithmetic
    assert sorted(np.concatenate(b1).tolist()) == list(range(23))          # each seed once
    b2 = Sa.epoch_batches(p, 5, 1, 4)
    assert not np.array_equal(np.concatenate(b1), np.concatenate(b2))      # reshuffled
    assert np.array_equal(np.concatenate(b1), np.concatenate(Sa.epoch_batches(p, 5, 0, 4)))


def test_conditional_uniformity():
    """over many independent draws each of d local neighbours is picked with
    frequency f/d (binomial, within 4 sigma)."""
    d, f, trials = 20, 5, 4000
    p = whole(d + 1, [(0, u) for u in range(1, d + 1)])
    counts = np.zeros(d + 1)
    for t in range(trials):
        b = Sa.sample_batch(p, [0], [f], 99, t, 0)[0]
        counts[b["src"][b["col"]]] += 1
    freq = counts[1:] / trials
    sigma = np.sqrt(f / d * (1 - f / d) / trials)
    assert np.all(np.abs(freq - f / d) <= 4 * sigma)
    assert counts.sum() == f * trials


def test_full_fanout_batch_equals_full_graph_layer():
    """One batch holding every node, fanout >= max degree: the block mean is the full local
    neighbourhood mean, so the seeds' logits equal oracle.model's full-graph SAGE layer."""
    rng = np.random.default_rng(1)
    n = 60
    edges = [(int(u), int(v)) for u, v in rng.integers(0, n, size=(150, 2))]
    p = whole(n, edges)
    X = rng.standard_normal((n, 5))
    Ws = [[rng.standard_normal((5, 3)), rng.standard_normal((5, 3))]]
    seeds = np.arange(n)
    blocks = Sa.sample_batch(p, seeds, [n], 3, 0, 0)
    lg, _ = Sa.sage_forward(blocks, X[blocks[0]["src"]], Ws)
    ref, _ = Mo.forward("sage", p["rowptr"], p["col"], X, Ws)
    assert np.max(np.abs(lg - ref[seeds])) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("depth", [2, 3])
def test_block_backward_finite_differences(depth):
    rng = np.random.default_rng(depth + 10)   # a draw with no pre-activation at a ReLU kink
    rp, col = gen.rmat(8, 200, 1500, 1, 2)
    p = Po.induced_partition(rp, col, Po.make_chunks(200, 2, 1), 0, 1, np.ones(200, np.uint8))
    fan = [4, 3, 2][-depth:]
    blocks = Sa.sample_batch(p, Sa.epoch_batches(p, 4, 0, 16)[0], fan, 4, 0, 0)
    X = rng.standard_normal((blocks[0]["n_src"], 4))
    y = rng.integers(0, 3, blocks[-1]["n_dst"])
    dims = [4] + [5] * (depth - 1) + [3]
    Ws = [[rng.standard_normal((dims[l], dims[l + 1])) * 0.7 for _ in range(2)] for l in range(depth)]
    seeds = np.arange(blocks[-1]["n_dst"])

    def loss(W):
        lg, cache = Sa.sage_forward(blocks, X, W)
        return Mo.loss_and_dlogits(lg, y, seeds), cache

    (L0, dZ), cache = loss(Ws)
    assert all(np.min(np.abs(Z)) > 1e-6 for Z in cache["Z"][:-1])
    g = Mo.flatten(Sa.sage_backward(blocks, cache, dZ, Ws))
    shapes = [[w.shape for w in ws] for ws in Ws]
    th = Mo.flatten(Ws)
    eps = 1e-6
    fd = np.array([(loss(Mo.unflatten(th + eps * e, shapes))[0][0] -
                    loss(Mo.unflatten(th - eps * e, shapes))[0][0]) / (2 * eps) for e in np.eye(th.size)])
    assert np.max(np.abs(fd - g)) / np.max(np.abs(fd)) <= 1e-5


def test_batch_correction_uses_hop1_sample_sizes():
    p = whole(6, [(0, 1), (0, 2), (0, 3), (0, 4), (1, 5)])
    blocks = Sa.sample_batch(p, [0, 1], [2], 1, 0, 0)
    d_l, d_g, s = Sa.batch_stats(p, blocks)
    assert d_l.tolist() == [4, 2] and s.tolist() == [2, 2]
    # eq:resampling with s_v: (4/4-1)*2 + (2/2-1)*2 = 0 -> guard -> 1
    assert Co.c_resampling(d_l, d_g, s) == 1.0


def test_floyd_subset_uniformity():
    """R24 (S:199 uniform without replacement): every f-subset of a target's d local neighbours
    is drawn equally often -- the subset law, not just the marginals (a range off by one in
    Floyd's step, t in [0, j) instead of [0, j], would skew it)."""
    from itertools import combinations
    d, f, trials = 6, 3, 8000
    p = whole(d + 1, [(0, u) for u in range(1, d + 1)])
    subsets = {c: 0 for c in combinations(range(1, d + 1), f)}
    for t in range(trials):
        b = Sa.sample_batch(p, [0], [f], 7, t, 0)[0]
        subsets[tuple(sorted(int(u) for u in b["src"][b["col"]]))] += 1
    assert sum(subsets.values()) == trials
    expect = trials / len(subsets)
    sigma = np.sqrt(expect * (1 - 1 / len(subsets)))
    assert all(abs(c - expect) <= 4 * sigma for c in subsets.values()), subsets
