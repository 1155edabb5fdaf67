"""Oracle step a10: isolated mini-batch sampling (config 4, sampling mode).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER: P:139 and P:177 (§3.2: "select a subset of the training nodes from the local partition
to construct subgraphs ... for a k-layer model we sample k-hop subgraphs"), P:382 (Alg. 1
isolated_sampling(partition)), P:489 (batch size 1000; fanouts {15,10,5} for 3 layers).
SPEC: S:196-204 (sample_batch: min(fanout, d_local) distinct local neighbours, uniform without
replacement), S:214-222 (epoch_iterator: shuffled core train nodes, batches of B, last smaller),
S:441/S:492 (lock-step iterations, shorter workers cycle their batches).

Readings:
  R23  epoch order: seeds sorted by (h(seed_s, epoch, gid(v)), gid(v)); batch b = slice b of B.
  R24  per target v at hop h with d = d_l(v) > f_h: f_h distinct neighbour positions drawn by
       Floyd's algorithm -- for j = d - f_h .. d - 1: r = h(h(seed_s, epoch, batch, h), gid(v), j),
       t = floor(r (j + 1) / 2^64) (uniform on [0, j]); keep t unless already kept, else keep j --
       a uniformly random f_h-subset, i.e. uniform without replacement; d <= f_h keeps all.
  R25  fanouts are listed input -> output layer, so hop 1 (the seeds' neighbours, the output
       layer) uses the LAST entry (5 of {15,10,5}) and hop L the first (Q17).
  R26  sources of hop h = targets of hop h (as a prefix, same order) followed by the newly
       reached nodes in ascending local id; each target's sampled sources listed in ascending
       source position.  Block l (input layer l = 1..L) is hop L-l+1.
  R27  SAGE on a block: h_out[v] = act(h_in[v] W_self + mean_{u in S(v)} h_in[u] W_nbr);
       mean over the SAMPLED set, 0 if empty.
  R28  batch correction uses the seeds' (d_l, d_g, s_v), s_v = hop-1 sample size.
"""
from __future__ import annotations

import numpy as np

from .partition import mix

M64 = (1 << 64) - 1


def _h(*args):
    acc = mix(np.asarray(args[-1], dtype=np.uint64))
    for a in reversed(args[:-1]):
        acc = mix(np.asarray(a, dtype=np.uint64) ^ acc)
    return acc


def epoch_batches(part, seed_s: int, epoch: int, B: int):
    """R23: the partition's seeds (local ids) in epoch order, cut into batches of B."""
    seeds = np.asarray(part["seeds"], dtype=np.int64)
    gid = np.asarray(part["core"], dtype=np.int64)[seeds]
    keys = _h(seed_s, epoch, gid)
    order = np.lexsort((gid, keys))
    s = seeds[order]
    return [s[i:i + B] for i in range(0, s.size, B)]


def sample_hop(part, targets, f: int, seed_s: int, epoch: int, batch: int, hop: int):
    """R24/R26 for one hop: returns (sources, block rowptr, block col = source positions)."""
    rowptr = np.asarray(part["rowptr"], dtype=np.int64)
    col = np.asarray(part["col"], dtype=np.int64)
    gid = np.asarray(part["core"], dtype=np.int64)
    key0 = _h(seed_s, epoch, batch, hop)
    picked = []
    for v in targets:
        nb = col[rowptr[v]:rowptr[v + 1]]
        d = nb.size
        if d > f:
            # Floyd's algorithm (R24): f distinct positions, every f-subset equally likely
            kept = []
            for j in range(d - f, d):
                r = int(_h(key0, np.uint64(gid[v]), np.uint64(j)))
                t = (r * (j + 1)) >> 64
                kept.append(j if t in kept else t)
            nb = nb[np.asarray(kept, dtype=np.int64)]
        picked.append(nb)
    tset = set(int(t) for t in targets)
    new = sorted(set(int(u) for p in picked for u in p) - tset)
    sources = np.concatenate([np.asarray(targets, dtype=np.int64), np.asarray(new, dtype=np.int64)])
    pos = {int(u): i for i, u in enumerate(sources)}
    brow = np.zeros(len(targets) + 1, dtype=np.int64)
    bcol = []
    for i, p in enumerate(picked):
        ps = sorted(pos[int(u)] for u in p)
        bcol.extend(ps)
        brow[i + 1] = brow[i] + len(ps)
    return sources, brow, np.asarray(bcol, dtype=np.int64)


def sample_batch(part, batch_seeds, fanouts, seed_s: int, epoch: int, batch: int):
    """Layered blocks for one batch.  fanouts listed input -> output layer (R25).
    Returns (blocks, node lists) with blocks[l] for input layer l = 0..L-1:
    dict(rowptr, col, n_src, n_dst); nodes[l] = local ids of layer l's sources."""
    L = len(fanouts)
    targets = np.asarray(batch_seeds, dtype=np.int64)
    hops = []
    for h in range(1, L + 1):
        f = fanouts[L - h]
        sources, brow, bcol = sample_hop(part, targets, f, seed_s, epoch, batch, h)
        hops.append(dict(rowptr=brow, col=bcol, n_dst=targets.size, n_src=sources.size,
                         dst=targets, src=sources))
        targets = sources
    return hops[::-1]          # blocks[0] = input layer = hop L


def block_operator(blk, node_w=None):
    """D_s^-1 A_block (mean over the sampled set; zero row if none) as a sparse matrix.
    node_w (node-level estimator, R30): per partition-local node weight d_l/d_g; target v's
    sampled mean is multiplied by node_w[v] (p/q with q = 1/d_l per draw, p = 1/d_g)."""
    import scipy.sparse as sp
    cnt = np.diff(blk["rowptr"]).astype(np.float64)
    rs = np.where(cnt > 0, 1.0 / np.maximum(cnt, 1), 0.0)
    if node_w is not None:
        rs = rs * np.asarray(node_w, dtype=np.float64)[np.asarray(blk["dst"], dtype=np.int64)]
    vals = np.repeat(rs, np.diff(blk["rowptr"]))
    return sp.csr_matrix((vals, blk["col"], blk["rowptr"]), shape=(blk["n_dst"], blk["n_src"]))


def sage_forward(blocks, X_src, weights, masks=None, node_w=None):
    """R27: SAGE over the blocks; X_src rows = blocks[0]['src'] (features of the outermost
    sources).  node_w: node-level estimator weights per local node (R30) or None.
    Returns (logits over the seeds, cache)."""
    H = np.asarray(X_src, dtype=np.float64)
    cache = dict(H=[], P=[], Z=[], M=[], ops=[])
    L = len(blocks)
    for l, (blk, Ws) in enumerate(zip(blocks, weights)):
        op = block_operator(blk, node_w)
        P = op @ H
        Z = H[:blk["n_dst"]] @ Ws[0] + P @ Ws[1]
        relu = l < L - 1
        mk = None if (masks is None or not relu) else masks[l]
        cache["H"].append(H); cache["P"].append(P); cache["Z"].append(Z); cache["ops"].append(op)
        cache["M"].append((Z > 0.0) if mk is None else mk)
        H = (np.maximum(Z, 0.0) if mk is None else Z * mk) if relu else Z
    return H, cache


def sage_backward(blocks, cache, dZ, weights):
    L = len(blocks)
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        H, P, op, Ws = cache["H"][l], cache["P"][l], cache["ops"][l], weights[l]
        nd = blocks[l]["n_dst"]
        grads[l] = [H[:nd].T @ dZ, P.T @ dZ]
        dH = op.T @ (dZ @ Ws[1].T)
        dH[:nd] += dZ @ Ws[0].T
        if l > 0:
            dZ = dH * cache["M"][l - 1]
    return grads


def batch_stats(part, blocks):
    """R28: (d_l, d_g, s_v) of the batch seeds (targets of the output block)."""
    out = blocks[-1]
    seeds = out["dst"]
    s = np.diff(out["rowptr"])
    return np.asarray(part["d_l"])[seeds], np.asarray(part["d_g"])[seeds], s
