"""Oracle steps a1-a3: chunking, sweep schedule, induced chunk-pair partition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

a1  P:194-198 (§3.3 "Chunks and Efficient Partition Construction"): nodes are randomly
    assigned to C chunks once.  Reading R1: chunk_of[v] = pi(v) mod C with pi a
    seeded 4-round Feistel bijection on [0,N) (cycle walking) -- SPEC's "uniform shuffled
    round-robin", balanced to +-1.
a2  P:207 ("Coverage guarantee"): worker w pins base chunk w and sweeps
    (w+t) mod C for t = 1..C-1 (W = C); reading R2 for W < C.
a3  P:198 + S:135-143 (induced-core mode): core = base u swept chunk, ascending
    global id; local id = rank; each core row keeps neighbours inside the core, ascending;
    d_l = kept count, d_g = global degree; seeds = core train nodes.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix(x):
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def h3(a, b, c):
    a = np.asarray(a, dtype=np.uint64)
    return mix(a ^ mix(np.asarray(b, dtype=np.uint64) ^ mix(np.asarray(c, dtype=np.uint64))))


def feistel_bits(n: int) -> int:
    lg = 0
    while (1 << lg) < n:
        lg += 1
    return max(2, 2 * ((lg + 1) // 2))


def feistel_pi(n: int, seed: int, v: np.ndarray) -> np.ndarray:
    """pi(v): 4-round balanced Feistel permutation of [0, 2^bits), cycle-walked into [0,n).
    Round r maps (L, R) -> (R, L ^ (h(seed, r, R) & mask))."""
    half = feistel_bits(n) // 2
    mask = np.uint64((1 << half) - 1)
    seed = np.uint64(seed)

    def once(x):
        L = x >> np.uint64(half)
        R = x & mask
        for r in range(4):
            L, R = R, L ^ (h3(seed, np.uint64(r), R) & mask)
        return (L << np.uint64(half)) | R

    y = once(np.asarray(v, dtype=np.uint64))
    bad = y >= np.uint64(n)
    while bad.any():
        y[bad] = once(y[bad])
        bad = y >= np.uint64(n)
    return y.astype(np.int64)


def make_chunks(n: int, C: int, seed: int) -> np.ndarray:
    """a1: chunk_of[v] = pi(v) mod C.  2 <= C <= n."""
    if not (2 <= C <= n):
        raise ValueError("need 2 <= C <= N (S:128)")
    return (feistel_pi(n, seed, np.arange(n, dtype=np.int64)) % C).astype(np.int32)


def sweep_schedule(C: int, W: int) -> list:
    """a2: list over super-epochs t = 1..cycle of [(base, swept)] per worker w = 0..W-1.

    W = C: pair(w, t) = (w, (w+t) mod C), cycle = C-1.
    W < C (reading R2): slot (t, w) -> unordered pair number ((t-1)*W + w) mod C(C-1)/2 in
    lexicographic order, base = lower chunk id; cycle = ceil(C(C-1) / (2W)).
    """
    if not (1 <= W <= C and C >= 2):
        raise ValueError("need 1 <= W <= C, C >= 2 (S:146)")
    if W == C:
        return [[(w, (w + t) % C) for w in range(W)] for t in range(1, C)]
    pairs = [(i, j) for i in range(C) for j in range(i + 1, C)]
    npairs = len(pairs)
    cycle = -(-npairs // W)
    return [[pairs[((t - 1) * W + w) % npairs] for w in range(W)] for t in range(1, cycle + 1)]


def pair_coverage(schedule: list, C: int) -> set:
    """Unordered chunk pairs NOT covered by the schedule."""
    covered = {frozenset(p) for row in schedule for p in row}
    return {frozenset((i, j)) for i in range(C) for j in range(i + 1, C)} - covered


def induced_partition(rowptr, col, chunk_of, base: int, swept: int, train=None, halo: bool = False):
    """a3: partition of chunks {base, swept}.

    induced-core (default): core = nodes of both chunks, each core row keeps the
    neighbours inside the core (cut edges dropped).
    halo-1 ("halo nodes ... cache boundary neighbors", "Should an endpoint not be
    part of the initial partition, it is incorporated as a halo node"; readings
    R33/R34): halo = {u not in core : u in N(v) for some core v}; every core row keeps ALL its
    neighbours (d_l = d_g), halo rows are empty (truncated adjacency, d_l = 0); local ids =
    core in ascending global id, then halo in ascending global id.

    Returns dict: core (global ids of ALL local nodes, core then halo), n_core, rowptr/col
    (local CSR over all local nodes, local ids listed in ascending GLOBAL id per row -- the
    same as ascending local id in induced-core mode), d_l, d_g (per local node),
    seeds (local ids of core train nodes, ascending)."""
    if base == swept:
        raise ValueError("base == swept (S:139)")
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    in_core = (chunk_of == base) | (chunk_of == swept)
    core = np.nonzero(in_core)[0]                       # ascending global id
    nodes = core
    if halo:
        reach = np.zeros(chunk_of.size, dtype=bool)
        for v in core:
            reach[col[rowptr[v]:rowptr[v + 1]]] = True
        nodes = np.concatenate([core, np.nonzero(reach & ~in_core)[0]])
    visible = np.zeros(chunk_of.size, dtype=bool)
    visible[nodes] = True
    local_of = np.full(chunk_of.size, -1, dtype=np.int64)
    local_of[nodes] = np.arange(nodes.size)
    d_g = (rowptr[nodes + 1] - rowptr[nodes]).astype(np.int64)
    lrow = [np.zeros(0, dtype=np.int64)] * nodes.size
    d_l = np.zeros(nodes.size, dtype=np.int64)
    for i, v in enumerate(core):                        # halo rows stay empty
        nb = col[rowptr[v]:rowptr[v + 1]]
        kept = nb[visible[nb]]                          # keeps ascending global order
        lrow[i] = local_of[kept]
        d_l[i] = kept.size
    lrowptr = np.zeros(nodes.size + 1, dtype=np.int64)
    np.cumsum(d_l, out=lrowptr[1:])
    lcol = np.concatenate(lrow) if nodes.size else np.zeros(0, dtype=np.int64)
    seeds = np.zeros(0, dtype=np.int64) if train is None else \
        np.nonzero(np.asarray(train)[core] != 0)[0]
    return dict(core=nodes, n_core=core.size, rowptr=lrowptr, col=lcol, d_l=d_l, d_g=d_g,
                seeds=seeds)
