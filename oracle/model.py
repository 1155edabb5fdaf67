"""Oracle steps a4-a6: k-layer GCN / GraphSAGE forward, softmax cross-entropy, backward.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything is float64, textbook order, on the partition-local CSR only (cut edges are
simply absent from it -- P:141, "considers exclusively local nodes and edges").

GCN layer ("averages neighbors with degree-based weights"; readings R5, R7):
    Z = Ahat H W,  Ahat = Dt^-1/2 (A + I) Dt^-1/2,  Dt = diag(d_l + 1)  (virtual self-loop)
SAGE layer ("aggregated (for example, by averaging) ... combined and multiplied by a
matrix"; reading R6):
    M = D_l^-1 A H  (row of zeros where d_l = 0),  Z = H W_self + M W_nbr
GAT layer ("assigns weights to different neighborhood nodes using attention ... modified
by a matrix (a linear layer) ... averaging its neighbors' hidden states using learned weights";
reading R35: one head, self loop, LeakyReLU 0.2, no bias):
    z = H W,  alpha_vu = softmax_{u in N(v)+v} LeakyReLU(z_u a_src + z_v a_dst),  Z = alpha z
    parameters per layer [W, [a_src; a_dst]]
Activation: ReLU on hidden layers, identity on the output layer; ReLU'(0) = 0 (R16).
No biases (R7).  Loss: mean softmax cross-entropy over the partition's seeds with a
max-subtracted log-sum-exp (R8).  Backward: exact reverse mode.
Parameters theta = concatenation in layer order of W (GCN) or W_self, W_nbr (SAGE), each
[d_in x d_out] row-major.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def adjacency(rowptr, col, n: int) -> sp.csr_matrix:
    """A (local, unweighted, symmetric) as a sparse matrix; A[v, u] = 1 iff u in N_loc(v)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    return sp.csr_matrix((np.ones(col.size, dtype=np.float64), col, rowptr), shape=(n, n))


def gcn_operator(rowptr, col, n: int, node_w=None) -> sp.csr_matrix:
    """Ahat = Dt^-1/2 (A + I) Dt^-1/2 with Dt = d_l + 1.
    node_w (node-level estimator, eq. (9), reading R30): target v's neighbour
    message is multiplied by w_v, the self term is not:  Dt^-1/2 (diag(w) A + I) Dt^-1/2."""
    A = adjacency(rowptr, col, n)
    if node_w is not None:
        A = sp.diags(np.asarray(node_w, dtype=np.float64)) @ A
    d_l = np.diff(np.asarray(rowptr, dtype=np.int64)).astype(np.float64)
    nrm = 1.0 / np.sqrt(d_l + 1.0)
    Dn = sp.diags(nrm)
    return (Dn @ (A + sp.identity(n, format="csr")) @ Dn).tocsr()


def sage_operator(rowptr, col, n: int, node_w=None) -> sp.csr_matrix:
    """D_l^-1 A (mean over local neighbours; zero row where d_l = 0).
    node_w (R30): the mean message of target v is multiplied by w_v:  diag(w) D_l^-1 A."""
    A = adjacency(rowptr, col, n)
    d_l = np.diff(np.asarray(rowptr, dtype=np.int64)).astype(np.float64)
    inv = np.where(d_l > 0, 1.0 / np.maximum(d_l, 1.0), 0.0)
    if node_w is not None:
        inv = inv * np.asarray(node_w, dtype=np.float64)
    return (sp.diags(inv) @ A).tocsr()


def layer_forward(arch: str, op, H, Ws, relu: bool, mask=None):
    """One layer: P = op H (Ahat H or D^-1 A H); Z = P W (gcn) or H W_self + P W_nbr (sage);
    returns (P, Z, act(Z)).  `mask` (optional, reading R16b): the ReLU decision 1[Z > 0]
    taken by the kernel under test in its own precision -- act(Z) = Z * mask -- so that a
    pre-activation within rounding of 0 does not make the two sides branch differently."""
    if arch == "gat":
        # GAT (R35): z = H W; alpha from (z a_src, z a_dst); Z = alpha z.  P carries the
        # cache (z, alpha, LeakyReLU') for the backward.
        z = H @ Ws[0]
        alpha, slope = gat_attention(op, z, Ws[1][0], Ws[1][1])
        Z = alpha @ z
        P = (z, alpha, slope)
    else:
        P = op @ H
        Z = P @ Ws[0] if arch == "gcn" else H @ Ws[0] + P @ Ws[1]
    if not relu:
        return P, Z, Z
    return P, Z, (np.maximum(Z, 0.0) if mask is None else Z * mask)


def layer_backward(arch: str, op, H, P, Ws, dZ):
    """Reverse mode of layer_forward given dL/dZ: returns (weight grads, dL/dH)."""
    if arch == "gat":
        z, alpha, slope = P
        a_src, a_dst = Ws[1][0], Ws[1][1]
        dz = alpha.T @ dZ                                  # through Z = alpha z
        rows = np.repeat(np.arange(alpha.shape[0]), np.diff(alpha.indptr))
        cols = alpha.indices
        dalpha = np.einsum("ij,ij->i", dZ[rows], z[cols])  # dL/dalpha_vu = dZ_v . z_u
        c = np.zeros(alpha.shape[0])
        np.add.at(c, rows, alpha.data * dalpha)            # softmax backward
        dpre = alpha.data * (dalpha - c[rows]) * slope     # through LeakyReLU
        ds = np.zeros(alpha.shape[0])
        dt = np.zeros(alpha.shape[0])
        np.add.at(ds, cols, dpre)                          # s_u enters every edge (v, u)
        np.add.at(dt, rows, dpre)                          # t_v enters every edge of row v
        dz = dz + np.outer(ds, a_src) + np.outer(dt, a_dst)
        return [H.T @ dz, np.stack([z.T @ ds, z.T @ dt])], dz @ Ws[0].T
    if arch == "gcn":
        return [P.T @ dZ], op.T @ (dZ @ Ws[0].T)
    return [H.T @ dZ, P.T @ dZ], dZ @ Ws[0].T + op.T @ (dZ @ Ws[1].T)


def gat_pattern(rowptr, col, n: int) -> sp.csr_matrix:
    """GAT's attention support A_loc + I (each target attends to its local neighbours and to
    itself, reading R35) as a 0/1 matrix with sorted indices."""
    A = adjacency(rowptr, col, n)
    M = (A + sp.identity(n, format="csr")).tocsr()
    M.sort_indices()
    M.data[:] = 1.0
    return M


LRELU_SLOPE = 0.2     # GAT's LeakyReLU negative slope (Velickovic et al., reading R35)


def gat_attention(pattern, z, a_src, a_dst):
    """alpha_vu = softmax_{u in N(v) + v} LeakyReLU(s_u + t_v), s = z a_src, t = z a_dst
    ("assigns weights to different neighborhood nodes using attention"; R35).  Returns
    (alpha as a sparse matrix on the pattern, LeakyReLU' per stored entry)."""
    s = z @ a_src
    t = z @ a_dst
    rows = np.repeat(np.arange(pattern.shape[0]), np.diff(pattern.indptr))
    cols = pattern.indices
    pre = s[cols] + t[rows]
    e = np.where(pre > 0, pre, LRELU_SLOPE * pre)
    slope = np.where(pre > 0, 1.0, LRELU_SLOPE)          # LeakyReLU'(0) = slope (R35)
    alpha = np.zeros_like(e)
    for v in range(pattern.shape[0]):                      # row-wise max-shifted softmax
        k0, k1 = pattern.indptr[v], pattern.indptr[v + 1]
        ev = e[k0:k1]
        w = np.exp(ev - ev.max())
        alpha[k0:k1] = w / w.sum()
    A = sp.csr_matrix((alpha, cols.copy(), pattern.indptr.copy()), shape=pattern.shape)
    return A, slope


def operator(arch: str, rowptr, col, n: int, node_w=None):
    if arch == "gat":
        if node_w is not None:
            raise ValueError("node-level weights are defined for mean/sum aggregators (R30), not GAT")
        return gat_pattern(rowptr, col, n)
    return (gcn_operator(rowptr, col, n, node_w) if arch == "gcn"
            else sage_operator(rowptr, col, n, node_w))


def forward(arch: str, rowptr, col, X, weights, masks=None, node_w=None):
    """Returns (logits, cache).  weights[l] = [W] (gcn) or [W_self, W_nbr] (sage), float64.
    masks (optional): per hidden layer the ReLU decision to use (see layer_forward).
    node_w (optional): node-level estimator weights, applied in every layer (R30)."""
    n = X.shape[0]
    op = operator(arch, rowptr, col, n, node_w)
    H = np.asarray(X, dtype=np.float64)
    cache = dict(op=op, H=[], P=[], Z=[], M=[])
    L = len(weights)
    for l, Ws in enumerate(weights):
        mk = None if masks is None or l >= L - 1 else masks[l]
        P, Z, Hn = layer_forward(arch, op, H, Ws, l < L - 1, mk)
        cache["H"].append(H); cache["P"].append(P); cache["Z"].append(Z)
        cache["M"].append((Z > 0.0) if mk is None else mk)
        H = Hn
    return H, cache


def loss_and_dlogits(Z, y, seeds):
    """L = (1/#S) sum_{v in S} [logsumexp(Z_v) - Z_v[y_v]];  dZ = (softmax - onehot)/#S on S."""
    seeds = np.asarray(seeds, dtype=np.int64)
    if seeds.size == 0:
        raise ValueError("empty seed set (S:213)")
    Zs = Z[seeds]
    m = Zs.max(axis=1, keepdims=True)
    e = np.exp(Zs - m)
    s = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(s))[:, 0]
    ys = np.asarray(y, dtype=np.int64)[seeds]
    if (ys >= Z.shape[1]).any() or (ys < 0).any():
        raise ValueError("label out of range (S:280)")
    loss = float(np.mean(lse - Zs[np.arange(seeds.size), ys]))
    dZ = np.zeros_like(Z, dtype=np.float64)
    g = e / s
    g[np.arange(seeds.size), ys] -= 1.0
    dZ[seeds] = g / seeds.size
    return loss, dZ


def backward(arch: str, cache, dlogits, weights):
    """Exact reverse mode through the cached forward; returns grads shaped like weights."""
    L = len(weights)
    grads = [None] * L
    dZ = dlogits
    for l in range(L - 1, -1, -1):
        grads[l], dH = layer_backward(arch, cache["op"], cache["H"][l], cache["P"][l],
                                      weights[l], dZ)
        if l > 0:
            dZ = dH * cache["M"][l - 1]                # ReLU' = 1[Z > 0], ReLU'(0) = 0 (R16)
    return grads


def flatten(mats) -> np.ndarray:
    return np.concatenate([np.asarray(m, dtype=np.float64).ravel() for ms in mats for m in ms])


def unflatten(theta, shapes) -> list:
    out, off = [], 0
    for ms in shapes:
        row = []
        for s in ms:
            k = int(np.prod(s))
            row.append(np.asarray(theta[off:off + k], dtype=np.float64).reshape(s))
            off += k
        out.append(row)
    return out


def partition_loss_grad(arch, part, X, y, weights, masks=None, node_w=None):
    """Loss L_p and flat gradient g_p of one isolated partition (full-graph mode).
    X is indexed by the partition's local ids (rows = part['core']).  node_w: per local node
    the node-level estimator weight (correction.node_weights), or None (batch-level kinds)."""
    logits, cache = forward(arch, part["rowptr"], part["col"], X, weights, masks, node_w)
    loss, dZ = loss_and_dlogits(logits, y, part["seeds"])
    grads = backward(arch, cache, dZ, weights)
    return loss, flatten(grads), logits, cache
