"""Pins for oracle steps a7-a9 (coverage factors, aggregation, SGD, Algorithm 1) -- CPU only.

Pins: SPEC.md hand values; full coverage -> 1; c_uniform in [0,1] and monotone; the HM
reading equals sum d_l / sum d_g in full-graph mode; Theorem 2: c_uniform is
the grid argmin of || E[corr] - c E[g] || built by explicit enumeration; the single-partition
case reduces to the ordinary full-graph gradient (dense re-derivation + finite differences);
uniform coverage gives the plain mean; finite differences of (1/M) sum_p c_p L_p(theta).
"""
import json
import math
import os

import numpy as np
import pytest

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as P
from oracle import train as Tr

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_values.json")))


def test_hand_values():
    for case in GOLD["c_uniform"]:
        assert math.isclose(Co.c_uniform(case["d_l"], case["d_g"]), case["c"], rel_tol=1e-15)
    for case in GOLD["c_resampling"]:
        assert Co.resampling_denominator(case["d_l"], case["d_g"], case["s"]) == case["D"]
        assert math.isclose(Co.c_resampling(case["d_l"], case["d_g"], case["s"]), case["c"],
                            rel_tol=1e-15)


def test_resampling_guards_and_integer_identity():
    assert Co.c_resampling([4], [4]) == 1.0                           # D = 0 < eps -> 1
    assert Co.c_resampling([20], [21], [1]) == Co.C_MAX               # D = 0.05 -> cap 10
    rng = np.random.default_rng(3)
    d_g = rng.integers(1, 50, 500)
    d_l = np.minimum(d_g, rng.integers(0, 50, 500))
    D_int = int(np.sum((d_g - d_l)[d_l > 0]))
    D_float = float(np.sum(((d_g / np.maximum(d_l, 1)) - 1.0)[d_l > 0] * d_l[d_l > 0]))
    assert Co.resampling_denominator(d_l, d_g) == float(D_int)
    assert math.isclose(D_float, D_int, rel_tol=1e-12)
    assert Co.c_resampling(d_l, d_g) == 1.0 / D_int


def test_uniform_properties():
    rng = np.random.default_rng(4)
    d_g = rng.integers(0, 30, 200)
    d_l = np.minimum(d_g, rng.integers(0, 30, 200))
    c = Co.c_uniform(d_l, d_g)
    assert 0.0 <= c <= 1.0
    assert Co.c_uniform(d_g, d_g) == 1.0                               # full coverage
    for i in np.nonzero(d_l < d_g)[0][:20]:                            # monotone
        d2 = d_l.copy(); d2[i] += 1
        assert Co.c_uniform(d2, d_g) >= c
    assert Co.c_uniform([0], [0]) == 1.0 and Co.c_uniform([0], [5]) == 0.0   # R4
    with pytest.raises(ValueError):
        Co.c_uniform([], [])


def test_hm_reading():
    rng = np.random.default_rng(5)
    d_g = rng.integers(1, 30, 300)
    d_l = np.minimum(d_g, rng.integers(0, 30, 300))
    k = d_l > 0
    assert math.isclose(Co.c_resampling_hm(d_l, d_g), d_l[k].sum() / d_g[k].sum(), rel_tol=1e-13)
    assert Co.c_resampling_hm(d_g, d_g) == 1.0
    # HM <= AM of r over the same (s-)weights
    r = d_l[k] / d_g[k]
    am = float(np.sum(d_l[k] * r) / np.sum(d_l[k]))
    assert Co.c_resampling_hm(d_l, d_g) <= am + 1e-15


@pytest.mark.parametrize("mu_dim", [1, 8, 64])
@pytest.mark.parametrize("dist", ["constant", "two_point", "uniform"])
def test_theorem2_projection(mu_dim, dist):
    """with g_v(u) = mu i.i.d., the minimiser of ||E[corr] - c E[g]|| is the batch
    factor (eq:batch_correction_factor); uniform p,q -> ratio d_l/d_g per neighbour."""
    rng = np.random.default_rng(mu_dim * 7 + len(dist))
    mu = rng.standard_normal(mu_dim) * 3
    nodes = 40
    d_g = rng.integers(2, 12, nodes)
    if dist == "constant":
        d_l = d_g.copy()
    elif dist == "two_point":
        d_l = np.where(np.arange(nodes) % 2 == 0, d_g, np.maximum(1, d_g // 2))
    else:
        d_l = np.maximum(1, (rng.uniform(0.1, 1.0, nodes) * d_g).astype(int))
    # E[corr] by explicit enumeration: (1/|S|) sum_v (1/|S_v|) sum_{u in S_v} p_v(u)/q_v(u) mu
    e_corr = np.zeros(mu_dim)
    for v in range(nodes):
        p, q = 1.0 / d_g[v], 1.0 / d_l[v]
        e_corr += sum((p / q) * mu for _ in range(d_l[v])) / d_l[v]
    e_corr /= nodes
    c_star = Co.c_uniform(d_l, d_g)
    grid = np.arange(0.0, 3 * c_star + 1e-3, 1e-3)
    obj = [np.linalg.norm(e_corr - c * mu) for c in grid]
    assert abs(grid[int(np.argmin(obj))] - c_star) <= 2e-3


def test_aggregate_identities():
    rng = np.random.default_rng(6)
    g = rng.standard_normal(50)
    assert np.allclose(Co.aggregate([1.0, 1.0], [g, -g], 2), 0.0)
    assert np.allclose(Co.aggregate([1.0] * 3, [g] * 3, 3), g)
    gs = [rng.standard_normal(50) for _ in range(4)]
    assert np.allclose(Co.aggregate([0.3] * 4, gs, 4), 0.3 * np.mean(gs, axis=0))
    with pytest.raises(FloatingPointError):
        Co.aggregate([1.0], [np.array([np.inf])], 1)
    th = rng.standard_normal(50)
    assert np.allclose(Co.sgd(Co.sgd(th, g, 0.0015), g, 0.0015), Co.sgd(th, g, 0.003))
    assert np.allclose(Co.sgd(th, th, 1.0), 0.0)


def _dense_full_graph_grad(n, edges, X, y, train_nodes, Ws):
    """Dense full-graph GCN loss/gradient over all train nodes (P:218-230 eq:gradient,
    S:519-527), re-derived with dense matrices -- shares nothing with oracle.model."""
    A = np.zeros((n, n))
    for u, v in edges:
        if u != v:
            A[u, v] = A[v, u] = 1.0
    At = A + np.eye(n)
    d = At.sum(1)
    Ah = At / np.sqrt(d)[:, None] / np.sqrt(d)[None, :]
    Hs, Zs = [X], []
    for l, W in enumerate(Ws):
        Z = Ah @ Hs[-1] @ W
        Zs.append(Z)
        Hs.append(np.maximum(Z, 0) if l < len(Ws) - 1 else Z)
    S = np.asarray(train_nodes)
    lg = Zs[-1][S]
    p = np.exp(lg - lg.max(1, keepdims=True)); p /= p.sum(1, keepdims=True)
    loss = float(np.mean(-np.log(p[np.arange(S.size), y[S]])))
    G = np.zeros_like(Zs[-1]); p[np.arange(S.size), y[S]] -= 1; G[S] = p / S.size
    grads = []
    for l in range(len(Ws) - 1, -1, -1):
        grads.append((Ah @ Hs[l]).T @ G)
        if l > 0:
            G = (Ah.T @ (G @ Ws[l].T)) * (Zs[l - 1] > 0)
    return loss, np.concatenate([g.ravel() for g in grads[::-1]])


@pytest.mark.parametrize("kind", ["none", "uniform", "resampling", "resampling_hm"])
def test_single_partition_is_full_graph_gradient(kind):
    """C = 2, W = 1: the one partition is the whole graph, every c = 1 and g_hat is the
    ordinary full-graph gradient."""
    n = 60
    rng = np.random.default_rng(7)
    edges = [(int(u), int(v)) for u, v in rng.integers(0, n, size=(150, 2))]
    rp, col = gen.csr_from_edges(n, edges)
    X = rng.standard_normal((n, 5)); y = rng.integers(0, 3, n)
    train = (rng.random(n) < 0.4).astype(np.uint8)
    Ws = [[rng.standard_normal((5, 4)) * 0.5], [rng.standard_normal((4, 3)) * 0.5]]
    ch = P.make_chunks(n, 2, 1)
    part = P.induced_partition(rp, col, ch, 0, 1, train)
    assert Tr.partition_factor(kind, part) == 1.0
    _, recs = Tr.run("gcn", rp, col, X, y, train, Ws, ch, 2, 1, 1, kind, 0.003, 1, 10)
    loss_ref, g_ref = _dense_full_graph_grad(n, edges, X, y, np.nonzero(train)[0],
                                             [w[0] for w in Ws])
    assert np.max(np.abs(recs[0]["g_hat"] - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
    assert math.isclose(recs[0]["loss"][0], loss_ref, rel_tol=1e-12)


def test_aggregated_update_finite_differences():
    """g_hat = grad of (1/M) sum_p c_p L_p(theta) with c_p fixed (a7)."""
    n = 40
    rng = np.random.default_rng(8)
    edges = [(int(u), int(v)) for u, v in rng.integers(0, n, size=(120, 2))]
    rp, col = gen.csr_from_edges(n, edges)
    X = rng.standard_normal((n, 4)); y = rng.integers(0, 3, n)
    train = (rng.random(n) < 0.5).astype(np.uint8)
    C, W, M = 4, 4, 4
    ch = P.make_chunks(n, C, 2)
    Ws = [[rng.standard_normal((4, 3)) * 0.7, rng.standard_normal((4, 3)) * 0.7]]
    _, recs = Tr.run("sage", rp, col, X, y, train, Ws, ch, C, W, M, "uniform", 0.003, 1, 10)
    parts = Tr.build_partitions(rp, col, ch, P.sweep_schedule(C, W)[0], train)
    cs = [Tr.partition_factor("uniform", p) for p in parts]
    assert cs == recs[0]["c"]
    shapes = [[w.shape for w in ws] for ws in Ws]
    theta = Mo.flatten(Ws)

    def F(t):
        tot = 0.0
        for c, p in zip(cs, parts):
            out, _ = Mo.forward("sage", p["rowptr"], p["col"], X[p["core"]], Mo.unflatten(t, shapes))
            tot += c * Mo.loss_and_dlogits(out, y[p["core"]], p["seeds"])[0]
        return tot / M

    eps = 1e-6
    fd = np.array([(F(theta + eps * e) - F(theta - eps * e)) / (2 * eps) for e in np.eye(theta.size)])
    assert np.max(np.abs(fd - recs[0]["g_hat"])) / np.max(np.abs(fd)) <= 1e-6


def test_phase_loop_structure():
    """Alg. 1: ceil(W/M) phases per epoch, one SGD step per phase, theta carried over."""
    n = 80
    rp, col = gen.rmat(7, n, 400, 1, 2)
    rng = np.random.default_rng(9)
    X = rng.standard_normal((n, 3)); y = rng.integers(0, 2, n)
    train = np.ones(n, dtype=np.uint8)
    Ws = [[rng.standard_normal((3, 2))]]
    ch = P.make_chunks(n, 4, 3)
    _, recs = Tr.run("gcn", rp, col, X, y, train, Ws, ch, 4, 4, 2, "none", 0.1, 3, 2)
    assert [r["phase"] for r in recs] == [0, 1] * 3
    assert [r["active"] for r in recs[:2]] == [[0, 1], [2, 3]]
    assert [r["t"] for r in recs] == [1, 1, 1, 1, 2, 2]                # repartition every 2
    th = Mo.flatten(Ws)
    for r in recs:
        th = th - 0.1 * r["g_hat"]
        assert np.allclose(th, r["theta"])
