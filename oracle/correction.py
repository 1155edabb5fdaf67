"""Oracle steps a7-a8: coverage correction factors, gradient aggregation, SGD.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Batch-level estimator (eq:batch-estimator): the partition's ordinary batch
gradient g_p is multiplied by one scalar c_p before the phase all-reduce (P:306,
Alg. 1).

  c_uniform    (eq:correction_uniform): (1/#S) sum_{v in S} d_l(v)/d_g(v);
               reading R4: d_l/d_g literal (0 allowed), ratio 1 iff d_g = 0.
  c_resampling (eq:resampling), literal with SPEC guards (R12):
               D = sum_{v in S, d_l>0} (d_g/d_l - 1) s_v ; c = 1 if D < eps else min(1/D, c_max)
               Full-graph mode (s_v = d_l): D = sum (d_g - d_l) is an integer -> c = 1/D.
  c_resampling_hm (optional reading R13, not the default): sum s_v / sum s_v d_g/d_l over
               v in S with d_l > 0; 1 if that set is empty.

Node-level estimator (eq. (4) and its uniform case eq. (9); SPEC S:321-329,
S:366-374; reading R30): every target v's neighbour contribution is importance-weighted by
p_v(u)/q_v^t(u).  Uniform neighbour distributions give p = 1/d_g, q = 1/d_l, i.e. one weight per
target w_v = d_l(v)/d_g(v) (1 iff d_g = 0, as R4); the weights enter the model as multipliers on
each target's aggregated neighbour message in every layer (oracle.model operators, node_w) and
the batch factor is then c_p = 1.

Aggregate (Alg. 1; R9): g_hat = (1/M) sum_{p active, ascending worker id}
c_p g_p; non-finite -> error.  SGD (lr = 0.003 P:489): theta - lr g_hat.
"""
from __future__ import annotations

import math

import numpy as np

EPS = 1e-9
C_MAX = 10.0


def c_uniform(d_l, d_g) -> float:
    d_l = np.asarray(d_l, dtype=np.int64)
    d_g = np.asarray(d_g, dtype=np.int64)
    if d_l.size == 0:
        raise ValueError("empty seed set (S:343)")
    r = np.where(d_g == 0, 1.0, d_l / np.where(d_g == 0, 1, d_g))
    return float(np.sum(r) / d_l.size)


def resampling_denominator(d_l, d_g, s=None) -> float:
    """D = sum_{v: d_l>0} (d_g/d_l - 1) * s_v (exact integer sum when s = d_l)."""
    d_l = np.asarray(d_l, dtype=np.int64)
    d_g = np.asarray(d_g, dtype=np.int64)
    s = d_l if s is None else np.asarray(s, dtype=np.int64)
    k = d_l > 0
    if s is d_l:
        return float(int(np.sum(d_g[k] - d_l[k])))   # (d_g/d_l - 1) d_l = d_g - d_l
    return float(np.sum((d_g[k] / d_l[k] - 1.0) * s[k]))


def c_resampling(d_l, d_g, s=None, eps: float = EPS, c_max: float = C_MAX) -> float:
    D = resampling_denominator(d_l, d_g, s)
    if D < eps:
        return 1.0
    return min(1.0 / D, c_max)


def c_resampling_hm(d_l, d_g, s=None) -> float:
    d_l = np.asarray(d_l, dtype=np.int64)
    d_g = np.asarray(d_g, dtype=np.int64)
    s = d_l if s is None else np.asarray(s, dtype=np.int64)
    k = d_l > 0
    if not k.any():
        return 1.0
    num = float(np.sum(s[k]))
    den = float(np.sum(s[k] * (d_g[k] / d_l[k])))
    return num / den


def coverage_factor(kind: str, d_l, d_g, s=None) -> float:
    if kind in ("none", "node"):      # node-level: the correction is inside the gradient
        return 1.0
    if kind == "uniform":
        return c_uniform(d_l, d_g)
    if kind == "resampling":
        return c_resampling(d_l, d_g, s)
    if kind == "resampling_hm":
        return c_resampling_hm(d_l, d_g, s)
    raise ValueError(kind)


def node_weight(p: float, q: float) -> float:
    """Importance weight p_v(u)/q_v^t(u) of one locally present neighbour (eq. (4));
    q = 0 violates Theorem 1's support condition."""
    if not q > 0.0:
        raise ValueError("support violation: q_v(u) = 0 (Theorem 1 precondition, S:325)")
    return p / q


def node_weights(d_l, d_g) -> np.ndarray:
    """Uniform special case (eq. (9)): w_v = p/q = (1/d_g)/(1/d_l) = d_l/d_g per target;
    1 where d_g = 0 (no neighbours at all, nothing to correct; R30)."""
    d_l = np.asarray(d_l, dtype=np.int64)
    d_g = np.asarray(d_g, dtype=np.int64)
    return np.where(d_g == 0, 1.0, d_l / np.where(d_g == 0, 1, d_g))


def importance_expectation(p_local, values) -> float:
    """Left side of the importance identity (eq. (3)) for a target whose local
    neighbours are drawn uniformly (q = 1/|local|): E_{u~q}[(p(u)/q(u)) g(u)], enumerated."""
    p_local = np.asarray(p_local, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    q = 1.0 / p_local.size
    return float(sum(q * node_weight(p, q) * g for p, g in zip(p_local, values)))


def aggregate(cs, grads, M: int) -> np.ndarray:
    """(1/M) sum_p c_p g_p, accumulated in ascending worker order."""
    out = np.zeros_like(np.asarray(grads[0], dtype=np.float64))
    for c, g in zip(cs, grads):
        if not math.isfinite(c):
            raise FloatingPointError("non-finite coverage factor (S:361)")
        out = out + c * np.asarray(g, dtype=np.float64)
    out = out / M
    if not np.all(np.isfinite(out)):
        raise FloatingPointError("non-finite gradient (S:424)")
    return out


def sgd(theta, g_hat, lr: float):
    return np.asarray(theta, dtype=np.float64) - lr * np.asarray(g_hat, dtype=np.float64)
