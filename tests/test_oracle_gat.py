"""Pins for the oracle's GAT layer (reading R35: one head, self loop,
LeakyReLU 0.2, no bias) -- CPU only.

Pins: attention written out by explicit per-node loops with math.exp (no sparse algebra);
zero attention vectors reduce to the plain mean over N(v) + v (closed form); an isolated node
attends only to itself; rows of alpha are probability vectors; central finite differences of
the loss through W and [a_src; a_dst] for depth 1 and 2, on a symmetric graph and on a halo-1
partition (non-symmetric)."""
import math

import numpy as np
import pytest

import gen
from oracle import model as Mo
from oracle import partition as P


def _graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    return gen.csr_from_edges(n, edges)


def test_attention_brute_force_loops():
    n = 15
    rp, col = _graph(n, 0.3, 1)
    rng = np.random.default_rng(2)
    H = rng.standard_normal((n, 4))
    W = rng.standard_normal((4, 3))
    a = rng.standard_normal((2, 3))
    _, Z, _ = Mo.layer_forward("gat", Mo.operator("gat", rp, col, n), H, [W, a], relu=False)
    z = H @ W
    for v in range(n):
        nb = sorted(list(col[rp[v]:rp[v + 1]]) + [v])
        e = []
        for u in nb:
            x = float(z[u] @ a[0] + z[v] @ a[1])
            e.append(x if x > 0 else 0.2 * x)
        m = max(e)
        w = [math.exp(x - m) for x in e]
        den = sum(w)
        ref = sum((wi / den) * z[u] for wi, u in zip(w, nb))
        assert np.allclose(Z[v], ref, rtol=1e-13, atol=1e-13)


def test_zero_attention_is_mean_and_isolated_node():
    rp, col = gen.csr_from_edges(6, [(0, 1), (1, 2), (0, 2), (2, 3)])   # nodes 4, 5 isolated
    rng = np.random.default_rng(3)
    H = rng.standard_normal((6, 5))
    W = rng.standard_normal((5, 4))
    op = Mo.operator("gat", rp, col, 6)
    _, Z, _ = Mo.layer_forward("gat", op, H, [W, np.zeros((2, 4))], relu=False)
    z = H @ W
    for v in range(6):
        nb = list(col[rp[v]:rp[v + 1]]) + [v]
        assert np.allclose(Z[v], z[nb].mean(axis=0), rtol=1e-14, atol=1e-14)
    _, Z2, _ = Mo.layer_forward("gat", op, H, [W, rng.standard_normal((2, 4))], relu=False)
    assert np.allclose(Z2[4:], z[4:], rtol=1e-15)                     # self-attention only
    alpha, _ = Mo.gat_attention(op, z, rng.standard_normal(4), rng.standard_normal(4))
    assert np.all(alpha.data >= 0) and np.allclose(np.asarray(alpha.sum(axis=1)).ravel(), 1.0)
    with pytest.raises(ValueError):
        Mo.operator("gat", rp, col, 6, node_w=np.ones(6))


@pytest.mark.parametrize("depth,halo", [(1, False), (2, False), (2, True)])
def test_gat_finite_differences(depth, halo):
    n = 30
    rp, col = _graph(n, 0.15, 4 + depth)
    rng = np.random.default_rng(5)
    if halo:
        ch = P.make_chunks(n, 5, 3)
        part = P.induced_partition(rp, col, ch, 0, 2, np.ones(n, np.uint8), halo=True)
        assert part["core"].size > part["n_core"]
    else:
        part = dict(rowptr=rp, col=col, seeds=np.arange(0, n, 2))
    m = part["rowptr"].size - 1
    X = rng.standard_normal((m, 3))
    y = rng.integers(0, 3, m)
    dims = [3] + [4] * (depth - 1) + [3]
    Ws = [[rng.standard_normal((dims[l], dims[l + 1])) * 0.8, rng.standard_normal((2, dims[l + 1]))]
          for l in range(depth)]
    _, g, _, cache = Mo.partition_loss_grad("gat", part, X, y, Ws)
    for Z in cache["Z"][:-1]:
        if np.min(np.abs(Z)) < 1e-4:
            pytest.skip("pre-activation near a ReLU kink")
    theta = Mo.flatten(Ws)
    shapes = [[w.shape for w in ws] for ws in Ws]
    num = np.zeros_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        num[i] = (Mo.partition_loss_grad("gat", part, X, y, Mo.unflatten(tp, shapes))[0] -
                  Mo.partition_loss_grad("gat", part, X, y, Mo.unflatten(tm, shapes))[0]) / 2e-6
    assert np.max(np.abs(num - g)) / np.max(np.abs(g)) <= 1e-5
