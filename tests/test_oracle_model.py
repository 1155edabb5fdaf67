"""Pins for oracle steps a4-a6 (GCN/SAGE forward, loss, backward) -- CPU only.

Pins: closed forms (d-regular GCN with H=1, W=I gives 1; SAGE mean of a constant; zero
weights; uniform logits -> ln K; the 2-node path 1/sqrt(2*2)), a dense adjacency-matrix
re-derivation on <= 200 nodes, and central finite differences.
"""
import json
import math
import os

import numpy as np
import pytest

import gen
from oracle import model as Mo

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_values.json")))


def ring(n, k):
    """circulant k-regular graph (k even): v ~ v +- 1..k/2"""
    return gen.csr_from_edges(n, [(v, (v + j) % n) for v in range(n) for j in range(1, k // 2 + 1)])


def test_gcn_regular_graph_gives_one():
    rp, col = ring(12, 4)
    X = np.ones((12, 3))
    W = [[np.eye(3)]]
    out, _ = Mo.forward("gcn", rp, col, X, W)
    assert np.allclose(out, 1.0, atol=1e-15, rtol=0)


def test_sage_mean_of_constant():
    rp, col = gen.csr_from_edges(5, [(0, 1), (1, 2), (0, 2)])   # nodes 3,4 isolated
    X = np.full((5, 2), 3.5)
    out, _ = Mo.forward("sage", rp, col, X, [[np.zeros((2, 2)), np.eye(2)]])
    assert np.allclose(out[:3], 3.5) and np.all(out[3:] == 0.0)


def test_two_node_path():
    rp, col = gen.csr_from_edges(2, [(0, 1)])
    op = Mo.gcn_operator(rp, col, 2).toarray()
    assert np.allclose(op, GOLD["gcn_two_node_path"]["entry"])
    out, _ = Mo.forward("gcn", rp, col, np.array([[2.0], [4.0]]), [[np.array([[1.0]])]])
    assert np.allclose(out, 3.0)


def test_zero_weights_zero_logits_and_closed_form_grad():
    rp, col = ring(10, 2)
    X = np.random.default_rng(0).standard_normal((10, 4))
    K = 3
    W = [[np.zeros((4, 5))], [np.zeros((5, K))]]
    logits, cache = Mo.forward("gcn", rp, col, X, W)
    assert np.all(logits == 0)
    y = np.arange(10) % K
    seeds = np.arange(10)
    loss, dZ = Mo.loss_and_dlogits(logits, y, seeds)
    assert math.isclose(loss, math.log(K), rel_tol=1e-15)
    # softmax-CE at uniform logits: dZ = (1/K - onehot)/#S
    expect = (np.full((10, K), 1.0 / K) - np.eye(K)[y]) / 10
    assert np.allclose(dZ, expect, atol=1e-16)


def test_loss_uniform_logits_golden():
    g = GOLD["loss_uniform_logits"]
    loss, _ = Mo.loss_and_dlogits(np.full((4, g["K"]), 0.7), np.array([0, 1, 2, 0]), [0, 1, 2, 3])
    assert math.isclose(loss, g["loss"], rel_tol=1e-15)


def test_param_count_golden():
    g = GOLD["param_count"]
    d = g["dims"]
    gcn = [[np.zeros((d[l], d[l + 1]))] for l in range(2)]
    sage = [[np.zeros((d[l], d[l + 1]))] * 2 for l in range(2)]
    assert Mo.flatten(gcn).size == g["gcn"] and Mo.flatten(sage).size == g["sage"]


def _dense_gcn_forward(n, edges, X, Ws):
    """Independent dense re-derivation: Dt^-1/2 (A+I) Dt^-1/2 H W with A from the edge list."""
    A = np.zeros((n, n))
    for u, v in edges:
        if u != v:
            A[u, v] = A[v, u] = 1.0
    At = A + np.eye(n)
    d = At.sum(1)
    Ah = At / np.sqrt(d)[:, None] / np.sqrt(d)[None, :]
    H = X
    for l, W in enumerate(Ws):
        Z = Ah @ H @ W
        H = np.maximum(Z, 0) if l < len(Ws) - 1 else Z
    return H


def _dense_sage_forward(n, edges, X, Ws):
    A = np.zeros((n, n))
    for u, v in edges:
        if u != v:
            A[u, v] = A[v, u] = 1.0
    deg = A.sum(1)
    H = X
    for l, (Wsf, Wn) in enumerate(Ws):
        Mn = np.zeros_like(H)
        for v in range(n):
            if deg[v] > 0:
                Mn[v] = A[v] @ H / deg[v]
        Z = H @ Wsf + Mn @ Wn
        H = np.maximum(Z, 0) if l < len(Ws) - 1 else Z
    return H


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_forward_matches_dense(arch, seed):
    rng = np.random.default_rng(seed)
    n = 150 + seed * 20
    edges = [(int(u), int(v)) for u, v in rng.integers(0, n, size=(4 * n, 2))]
    rp, col = gen.csr_from_edges(n, edges)
    dims = [7, 6, 5, 3]
    X = rng.standard_normal((n, dims[0]))
    Ws = [[rng.standard_normal((dims[l], dims[l + 1])) for _ in range(1 if arch == "gcn" else 2)]
          for l in range(3)]
    out, _ = Mo.forward(arch, rp, col, X, Ws)
    ref = (_dense_gcn_forward(n, edges, X, [w[0] for w in Ws]) if arch == "gcn"
           else _dense_sage_forward(n, edges, X, Ws))
    assert np.max(np.abs(out - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def _fd_case(arch, depth, seed):
    """10-node graph, theta chosen so no hidden pre-activation lies within 1e-4 of 0."""
    n = 10
    rng = np.random.default_rng(1000 + seed)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.35]
    rp, col = gen.csr_from_edges(n, edges)
    dims = [4] + [5] * (depth - 1) + [3]
    X = rng.standard_normal((n, 4))
    y = rng.integers(0, 3, n)
    seeds = np.array([0, 2, 3, 5, 7, 8])
    for _ in range(100):
        Ws = [[rng.standard_normal((dims[l], dims[l + 1])) * 0.8
               for _ in range(1 if arch == "gcn" else 2)] for l in range(depth)]
        _, cache = Mo.forward(arch, rp, col, X, Ws)
        if all(np.min(np.abs(Z)) > 1e-4 for Z in cache["Z"][:-1]):
            return rp, col, X, y, seeds, Ws
    raise RuntimeError("no valid theta")


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_backward_finite_differences(arch, depth):
    rp, col, X, y, seeds, Ws = _fd_case(arch, depth, depth)
    logits, cache = Mo.forward(arch, rp, col, X, Ws)
    _, dZ = Mo.loss_and_dlogits(logits, y, seeds)
    g = Mo.flatten(Mo.backward(arch, cache, dZ, Ws))
    shapes = [[w.shape for w in ws] for ws in Ws]
    theta = Mo.flatten(Ws)

    def f(t):
        out, _ = Mo.forward(arch, rp, col, X, Mo.unflatten(t, shapes))
        return Mo.loss_and_dlogits(out, y, seeds)[0]

    eps = 1e-6
    fd = np.zeros_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += eps; tm[i] -= eps
        fd[i] = (f(tp) - f(tm)) / (2 * eps)
    err = np.max(np.abs(g - fd)) / np.max(np.abs(fd))
    assert err <= 1e-5, err


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_given_masks_equal_own_decisions(arch):
    """R16b: passing the oracle's own ReLU decisions reproduces the default path exactly,
    and a flipped decision changes the gradient only through that unit."""
    rp, col, X, y, seeds, Ws = _fd_case(arch, 3, 9)
    logits, cache = Mo.forward(arch, rp, col, X, Ws)
    own = [(Z > 0).astype(np.float64) for Z in cache["Z"][:-1]]
    l2, c2 = Mo.forward(arch, rp, col, X, Ws, own)
    assert np.array_equal(logits, l2)
    _, dZ = Mo.loss_and_dlogits(logits, y, seeds)
    g1 = Mo.flatten(Mo.backward(arch, cache, dZ, Ws))
    g2 = Mo.flatten(Mo.backward(arch, c2, dZ, Ws))
    assert np.array_equal(g1, g2)


def test_empty_seed_and_bad_label():
    with pytest.raises(ValueError):
        Mo.loss_and_dlogits(np.zeros((3, 2)), np.zeros(3, int), [])
    with pytest.raises(ValueError):
        Mo.loss_and_dlogits(np.zeros((3, 2)), np.array([0, 2, 1]), [0, 1])


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_halo1_partition_finite_differences(arch):
    """halo-1 partitions make the local operator non-symmetric (core rows see halo nodes, halo
    rows are empty): the backward must use the transpose.  Central differences of the loss over
    the core seeds vs the reverse-mode gradient, depth 2."""
    from oracle import partition as P
    n = 40
    rng = np.random.default_rng(3)
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < 0.1]
    rp, col = gen.csr_from_edges(n, edges)
    ch = P.make_chunks(n, 5, 17)
    part = P.induced_partition(rp, col, ch, 1, 3, np.ones(n, np.uint8), halo=True)
    assert part["core"].size > part["n_core"]                 # there is a halo
    m = part["core"].size
    X = rng.standard_normal((m, 3))
    y = rng.integers(0, 3, m)
    nm = 1 if arch == "gcn" else 2
    Ws = [[rng.standard_normal((3, 4)) for _ in range(nm)], [rng.standard_normal((4, 3)) for _ in range(nm)]]
    L0, g, _, cache = Mo.partition_loss_grad(arch, part, X, y, Ws)
    if np.min(np.abs(cache["Z"][0])) < 1e-4:
        pytest.skip("pre-activation near a ReLU kink")
    op = cache["op"].toarray()
    assert not np.allclose(op, op.T)
    theta = Mo.flatten(Ws)
    shapes = [[w.shape for w in ws] for ws in Ws]
    num = np.zeros_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        num[i] = (Mo.partition_loss_grad(arch, part, X, y, Mo.unflatten(tp, shapes))[0] -
                  Mo.partition_loss_grad(arch, part, X, y, Mo.unflatten(tm, shapes))[0]) / 2e-6
    assert np.max(np.abs(num - g)) / np.max(np.abs(g)) <= 1e-5
