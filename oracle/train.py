"""Oracle step a9: Algorithm 1 (phase-parallel training) with super-epoch repartitioning.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Alg. 1: for each epoch, for phase i = 1..ceil(P/M): the active partitions
(workers [(i-1)M, iM)) each compute their isolated gradient (full-graph mode: the whole
partition), scale it by c_p, the scaled gradients are averaged over the
active workers and one optimizer step is taken; theta is carried to the
next phase.  Super-epochs: the partition layout is fixed for
`repartition_every` epochs, then every worker moves to the next swept chunk of the sweep
schedule (a2).  kind "node" = the node-level estimator (eq. (9), R30): per-target weights
d_l/d_g inside every layer's aggregation, c_p = 1.  Reading R11: one iteration per phase in full-graph mode.
"""
from __future__ import annotations

import numpy as np

from . import correction, model, partition


def build_partitions(rowptr, col, chunk_of, pairs, train):
    return [partition.induced_partition(rowptr, col, chunk_of, b, s, train) for (b, s) in pairs]


def partition_factor(kind, part):
    seeds = part["seeds"]
    return correction.coverage_factor(kind, part["d_l"][seeds], part["d_g"][seeds])


def run(arch, rowptr, col, X, y, train, weights, chunk_of, C, W, M, kind, lr, epochs,
        repartition_every, t0: int = 1, log=None):
    """Returns (final weights, list of per-step records).  weights: list of [W] / [Ws, Wn]."""
    sched = partition.sweep_schedule(C, W)
    shapes = [[w.shape for w in ws] for ws in weights]
    theta = model.flatten(weights)
    records = []
    parts, cur_t = None, None
    for e in range(epochs):
        t = t0 + e // repartition_every
        if t != cur_t:
            parts = build_partitions(rowptr, col, chunk_of, sched[(t - 1) % len(sched)], train)
            cur_t = t
        nphase = -(-W // M)
        for i in range(nphase):
            active = list(range(i * M, min((i + 1) * M, W)))
            Ws = model.unflatten(theta, shapes)
            cs, gs, losses = [], [], []
            for w in active:
                p = parts[w]
                Xp = np.asarray(X, dtype=np.float64)[p["core"]]
                yp = np.asarray(y)[p["core"]]
                nw = correction.node_weights(p["d_l"], p["d_g"]) if kind == "node" else None
                loss, g, _, _ = model.partition_loss_grad(arch, p, Xp, yp, Ws, node_w=nw)
                cs.append(partition_factor(kind, p)); gs.append(g); losses.append(loss)
            g_hat = correction.aggregate(cs, gs, len(active))
            theta = correction.sgd(theta, g_hat, lr)
            records.append(dict(epoch=e, t=t, phase=i, active=active, c=cs, loss=losses,
                                g_hat=g_hat, theta=theta.copy()))
    return model.unflatten(theta, shapes), records
