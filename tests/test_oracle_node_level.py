"""Pins for the oracle's node-level estimator -- CPU only.

PAPER §3.4: importance identity eq. (3), node-level estimator eq. (4) with
Theorem 1, uniform special case eq. (9) (p = 1/d_g, q = 1/d_l, weight
d_l/d_g per target).  SPEC S:321-329 (node_weight), S:366-374 (apply_node_level),
S:546-551 (verify_importance_identity).  Reading R30: the weight multiplies
every target's aggregated neighbour message in every layer; GCN's self term is unweighted.

Pins: SPEC's printed hand values; exact enumeration of the importance identity up to
d_global = 8; the first step of Theorem 1's proof (expectation over i.i.d. local draws),
enumerated exactly; brute-force per-node loops for the weighted
GCN / SAGE layers (no sparse algebra); closed forms (SAGE mean of a constant = coverage ratio,
weights 1 = the uncorrected model, zero-weight softmax gradient scales the neighbour path
only); central finite differences of the weighted model; and the long-run weighting the
deterministic sweep schedule actually gives (R31), enumerated over one full cycle.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import sampler as Sa

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_values.json")))


def test_node_weight_hand_values():
    for case in GOLD["node_weight"]:
        assert math.isclose(Co.node_weight(case["p"], case["q"]), case["w"], rel_tol=1e-15)
    with pytest.raises(ValueError):
        Co.node_weight(0.3, 0.0)                                  # support violation
    # uniform special case d_l/d_g (eq. (9)); d_g = 0 -> 1 (R30)
    w = Co.node_weights([1, 4, 0, 0, 3], [5, 4, 0, 7, 6])
    assert np.array_equal(w, np.array([0.2, 1.0, 1.0, 0.0, 0.5]))


def test_importance_identity_golden_and_enumerated():
    g = GOLD["importance_identity"]
    p = [1.0 / g["d_global"]] * len(g["local_values"])
    assert math.isclose(Co.importance_expectation(p, g["local_values"]), g["lhs"], rel_tol=1e-15)
    rng = np.random.default_rng(0)
    for d in range(1, 9):                                        # up to d_global = 8
        vals = rng.standard_normal(d)
        for k in range(1, d + 1):
            for sub in itertools.combinations(range(d), k):
                sub = list(sub)
                lhs = Co.importance_expectation([1.0 / d] * k, vals[sub])
                assert abs(lhs - np.sum(vals[sub]) / d) <= 1e-12 * (1 + np.abs(vals).sum())
        # full support: the ordinary expectation under p
        assert math.isclose(Co.importance_expectation([1.0 / d] * d, vals), float(np.mean(vals)),
                            rel_tol=1e-12, abs_tol=1e-15)


def test_estimator_expectation_over_iid_draws():
    """Theorem 1's proof, first step: with |S_v| = k i.i.d. draws u ~ D_v^local
    (uniform over the local set L, q = 1/d_l), the eq. (9)-weighted sample mean
    (1/k) sum_i (d_l/d_g) g_v(u_i) has expectation (1/d_g) sum_{u in L} g_v(u) = sum_{u in L}
    p_v(u) g_v(u) -- enumerated exactly over all d_l^k draw tuples -- and with L = N(v) (full
    support) it is E_{u ~ D_v}[g_v(u)], eq. (1)'s inner expectation.  The unweighted sample
    mean is off by d_g/d_l whenever L is a strict subset."""
    rng = np.random.default_rng(1)
    for d_g in range(1, 6):
        g = rng.standard_normal((d_g, 3))
        for d_l in range(1, d_g + 1):
            L = sorted(rng.choice(d_g, d_l, replace=False))
            w = Co.node_weights([d_l], [d_g])[0]
            for k in (1, 2, 3):
                tuples = list(itertools.product(L, repeat=k))
                est = np.mean([w * g[list(t)].mean(axis=0) for t in tuples], axis=0)
                assert np.allclose(est, g[L].sum(axis=0) / d_g, rtol=0, atol=1e-12)
                if d_l == d_g:
                    assert np.allclose(est, g.mean(axis=0), rtol=0, atol=1e-12)
                raw = np.mean([g[list(t)].mean(axis=0) for t in tuples], axis=0)
                assert np.allclose(raw * w, est, rtol=0, atol=1e-12)


def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    return gen.csr_from_edges(n, edges)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_weighted_layer_brute_force(arch):
    """per-node loops, no sparse algebra: GCN z_v = n_v (n_v h_v + w_v sum_u n_u h_u),
    SAGE z_v = h_v Ws + (w_v/d_l sum_u h_u) Wn (0 if d_l = 0)."""
    n = 30
    rp, col = _random_graph(n, 0.15, 3)
    rng = np.random.default_rng(4)
    H = rng.standard_normal((n, 5))
    w = rng.uniform(0.1, 1.0, n)
    Ws = [rng.standard_normal((5, 4)) for _ in range(1 if arch == "gcn" else 2)]
    _, Z, _ = Mo.layer_forward(arch, Mo.operator(arch, rp, col, n, w), H, Ws, relu=False)
    for v in range(n):
        nb = col[rp[v]:rp[v + 1]]
        d = len(nb)
        if arch == "gcn":
            nv = 1.0 / math.sqrt(d + 1)
            acc = nv * H[v]
            for u in nb:
                acc = acc + w[v] * H[u] / math.sqrt(rp[u + 1] - rp[u] + 1)
            ref = (nv * acc) @ Ws[0]
        else:
            m = np.zeros(5)
            for u in nb:
                m = m + H[u]
            m = m * (w[v] / d) if d > 0 else m
            ref = H[v] @ Ws[0] + m @ Ws[1]
        assert np.allclose(Z[v], ref, rtol=1e-13, atol=1e-13)


def test_sage_node_level_mean_of_constant_is_coverage_ratio():
    """SAGE with weights d_l/d_g: the corrected mean of a constant c is c d_l/d_g (the local
    sum divided by the GLOBAL degree), 0 where d_l = 0."""
    rp, col = gen.csr_from_edges(5, [(0, 1), (1, 2), (0, 2)])     # local graph
    d_l = np.diff(rp)
    d_g = np.array([4, 2, 3, 0, 5])
    X = np.full((5, 2), 3.0)
    out, _ = Mo.forward("sage", rp, col, X, [[np.zeros((2, 2)), np.eye(2)]],
                        node_w=Co.node_weights(d_l, d_g))
    assert np.allclose(out[:, 0], [3.0 * 2 / 4, 3.0 * 2 / 2, 3.0 * 2 / 3, 0.0, 0.0], rtol=1e-15)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_full_coverage_weights_one_is_uncorrected(arch):
    """C = 2 with one partition holding the whole graph: every d_l = d_g, all weights 1, the
    node-level gradient equals the uncorrected one (to 1e-14, the sparse product order
    may differ)."""
    rp, col = _random_graph(25, 0.2, 5)
    chunk_of = Po.make_chunks(25, 2, 9)
    part = Po.induced_partition(rp, col, chunk_of, 0, 1, np.ones(25, bool))
    w = Co.node_weights(part["d_l"], part["d_g"])
    assert np.all(w == 1.0)
    rng = np.random.default_rng(6)
    X = rng.standard_normal((25, 4))
    y = rng.integers(0, 3, 25)
    Ws = [[rng.standard_normal((4, 6)) for _ in range(1 if arch == "gcn" else 2)],
          [rng.standard_normal((6, 3)) for _ in range(1 if arch == "gcn" else 2)]]
    a = Mo.partition_loss_grad(arch, part, X, y, Ws, node_w=w)[1]
    b = Mo.partition_loss_grad(arch, part, X, y, Ws)[1]
    assert np.max(np.abs(a - b)) <= 1e-14 * np.max(np.abs(b))


def test_common_weight_scales_neighbour_path_only():
    """1-layer SAGE at zero weights (uniform logits, so dZ does not depend on
    w), every target with the same weight w: dW_nbr = w * uncorrected dW_nbr, dW_self
    unchanged (hand differentiation: Z = H Ws + w M Wn)."""
    rp, col = _random_graph(20, 0.25, 7)
    part = dict(rowptr=rp, col=col, seeds=np.arange(0, 20, 2))
    rng = np.random.default_rng(8)
    X = rng.standard_normal((20, 5))
    y = rng.integers(0, 4, 20)
    Ws = [[np.zeros((5, 4)), np.zeros((5, 4))]]
    _, g1, _, _ = Mo.partition_loss_grad("sage", part, X, y, Ws)
    _, gw, _, _ = Mo.partition_loss_grad("sage", part, X, y, Ws, node_w=np.full(20, 0.3))
    assert np.allclose(gw[:20], g1[:20], rtol=0, atol=1e-15)          # self path
    assert np.allclose(gw[20:], 0.3 * g1[20:], rtol=1e-13, atol=1e-16)  # neighbour path
    assert np.abs(g1[20:]).max() > 0


@pytest.mark.parametrize("arch,depth", [("gcn", 1), ("gcn", 3), ("sage", 1), ("sage", 2)])
def test_node_level_finite_differences(arch, depth):
    """central differences (eps 1e-6, f64) of the node-level weighted loss vs the reverse mode
    gradient; theta chosen away from ReLU kinks."""
    n = 12
    rp, col = _random_graph(n, 0.3, 10 + depth)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((n, 3))
    y = rng.integers(0, 3, n)
    w = rng.uniform(0.2, 1.0, n)
    dims = [3] + [4] * (depth - 1) + [3]
    nm = 1 if arch == "gcn" else 2
    Ws = [[rng.standard_normal((dims[l], dims[l + 1])) for _ in range(nm)] for l in range(depth)]
    part = dict(rowptr=rp, col=col, seeds=np.arange(n))
    _, g, _, cache = Mo.partition_loss_grad(arch, part, X, y, Ws, node_w=w)
    for Z in cache["Z"][:-1]:
        if np.min(np.abs(Z)) < 1e-4:
            pytest.skip("pre-activation too close to a ReLU kink")
    theta = Mo.flatten(Ws)
    shapes = [[m.shape for m in ms] for ms in Ws]
    eps = 1e-6
    num = np.zeros_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += eps; tm[i] -= eps
        lp = Mo.partition_loss_grad(arch, part, X, y, Mo.unflatten(tp, shapes), node_w=w)[0]
        lm = Mo.partition_loss_grad(arch, part, X, y, Mo.unflatten(tm, shapes), node_w=w)[0]
        num[i] = (lp - lm) / (2 * eps)
    assert np.max(np.abs(num - g)) / np.max(np.abs(g)) <= 1e-5


def test_minibatch_block_weights_brute_force():
    """mini-batch SAGE block with node-level weights: target v's SAMPLED mean times d_l/d_g."""
    rp, col = _random_graph(40, 0.2, 12)
    chunk_of = Po.make_chunks(40, 4, 13)
    part = Po.induced_partition(rp, col, chunk_of, 0, 2, np.ones(40, bool))
    w = Co.node_weights(part["d_l"], part["d_g"])
    seeds = np.asarray(part["seeds"])[:6]
    blocks = Sa.sample_batch(part, seeds, [3, 2], 21, 0, 0)
    op = Sa.block_operator(blocks[-1], w).toarray()
    blk = blocks[-1]
    for i, v in enumerate(blk["dst"]):
        c = blk["col"][blk["rowptr"][i]:blk["rowptr"][i + 1]]
        row = np.zeros(blk["n_src"])
        for j in c:
            row[j] += w[v] / len(c)
        assert np.allclose(op[i], row, rtol=1e-15, atol=0)


def test_sweep_long_run_weighting():
    """R31 (what the deterministic sweep gives, P:207 + eq. (9)): for per-edge contributions
    g_v(u), the average over the C-1 partitions of one cycle that hold v of
    (1/d_l) sum_{u local} (d_l/d_g) g_v(u) equals (1/d_g)(sum_{u same chunk} g_v(u)
    + (1/(C-1)) sum_{u other chunk} g_v(u)): neighbours in v's own chunk co-reside with v in
    every partition, cross-chunk neighbours in one of C-1, so eq. (9) is exact per partition
    (importance identity) but the cycle average over-weights same-chunk neighbours by C-1."""
    n, C = 36, 4
    rp, col = _random_graph(n, 0.2, 14)
    chunk_of = Po.make_chunks(n, C, 15)
    rng = np.random.default_rng(16)
    g = {}
    for v in range(n):
        for u in col[rp[v]:rp[v + 1]]:
            g[(v, int(u))] = rng.standard_normal()
    acc = np.zeros(n)
    cnt = np.zeros(n)
    sched = Po.sweep_schedule(C, C)
    for pairs in sched:
        for (b, s) in pairs:
            part = Po.induced_partition(rp, col, chunk_of, b, s)
            core = np.asarray(part["core"])
            w = Co.node_weights(part["d_l"], part["d_g"])
            for i, v in enumerate(core):
                loc = core[part["col"][part["rowptr"][i]:part["rowptr"][i + 1]]]
                if chunk_of[v] != b:
                    continue                      # count each (worker, t) once per base node
                dl = len(loc)
                acc[v] += (w[i] / dl) * sum(g[(int(v), int(u))] for u in loc) if dl else 0.0
                cnt[v] += 1
    for v in range(n):
        nb = col[rp[v]:rp[v + 1]]
        if len(nb) == 0:
            continue
        same = sum(g[(v, int(u))] for u in nb if chunk_of[u] == chunk_of[v])
        other = sum(g[(v, int(u))] for u in nb if chunk_of[u] != chunk_of[v])
        assert cnt[v] == C - 1
        assert math.isclose(acc[v] / cnt[v], (same + other / (C - 1)) / len(nb), rel_tol=1e-12,
                            abs_tol=1e-14)
