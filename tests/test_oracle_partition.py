"""Pins for oracle steps a1-a3 (chunking, schedule, induced partition) -- CPU only.

Each test ties the oracle to something other than itself: SPEC.md hand values
(tests/golden/spec_hand_values.json), brute force on tiny graphs, an independent
implementation of the same counter-based bijection (gen.scramble, C), the chunk-pair
edge-count identity and the one-cycle edge cover.
"""
import itertools
import json
import os

import numpy as np
import pytest

import gen
from oracle import partition as P

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_values.json")))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 17, 100, 1000, 4097])
def test_feistel_is_bijection(n):
    y = P.feistel_pi(n, 12345, np.arange(n))
    assert sorted(y.tolist()) == list(range(n))


@pytest.mark.parametrize("n,seed", [(10, 1), (2708, gen.seed_of("chunks")), (169343, 7)])
def test_feistel_matches_independent_c_implementation(n, seed):
    ids = np.arange(n, dtype=np.int64)
    assert np.array_equal(P.feistel_pi(n, seed, ids), gen.scramble(n, seed, ids))


@pytest.mark.parametrize("n,C", [(6, 3), (7, 2), (2708, 4), (10007, 8), (5, 5)])
def test_chunk_sizes_balanced(n, C):
    ch = P.make_chunks(n, C, 99)
    sizes = np.bincount(ch, minlength=C)
    assert sizes.sum() == n and sizes.max() - sizes.min() <= 1
    if (n, C) == (GOLD["chunk_sizes"]["n"], GOLD["chunk_sizes"]["C"]):
        assert sorted(sizes.tolist()) == GOLD["chunk_sizes"]["sizes"]
    if C == n:
        assert sizes.tolist() == [1] * n                                # S:133 singletons


def test_chunk_args():
    with pytest.raises(ValueError):
        P.make_chunks(5, 1, 0)
    with pytest.raises(ValueError):
        P.make_chunks(5, 6, 0)


def test_schedule_c3_hand_example():
    g = GOLD["schedule_C3"]
    sched = P.sweep_schedule(g["C"], g["W"])
    assert [[list(p) for p in row] for row in sched] == g["pairs"]


@pytest.mark.parametrize("C", range(2, 9))
def test_schedule_coverage_exhaustive(C):
    for W in range(1, C + 1):
        sched = P.sweep_schedule(C, W)
        assert P.pair_coverage(sched, C) == set(), (C, W)
        for row in sched:
            assert len(row) == W and all(b != s for b, s in row)
        if W < C:
            assert len(sched) == -(-C * (C - 1) // (2 * W))


def test_pair_coverage_detects_missing():
    assert P.pair_coverage([[(0, 1), (2, 3)]], 4) == {frozenset(p) for p in
                                                     [(0, 2), (0, 3), (1, 2), (1, 3)]}


def test_triangle_hand_example():
    g = GOLD["triangle_partition"]
    rp, col = gen.csr_from_edges(g["n"], g["edges"])
    part = P.induced_partition(rp, col, np.array(g["chunk_of"]), g["base"], g["swept"])
    assert part["core"].tolist() == g["core"]
    assert part["d_l"].tolist() == g["d_l"] and part["d_g"].tolist() == g["d_g"]
    assert part["col"].tolist() == [1, 0]


def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p]
    return edges


@pytest.mark.parametrize("seed", range(6))
def test_induced_partition_brute_force(seed):
    n = 23
    edges = _random_graph(n, 0.25, seed)
    rp, col = gen.csr_from_edges(n, edges)
    C = 4
    ch = P.make_chunks(n, C, seed + 100)
    train = (np.arange(n) % 3 == 0).astype(np.uint8)
    Adense = np.zeros((n, n), dtype=int)
    for u, v in edges:
        Adense[u, v] = Adense[v, u] = 1
    for b, s in itertools.permutations(range(C), 2):
        part = P.induced_partition(rp, col, ch, b, s, train)
        core = [v for v in range(n) if ch[v] in (b, s)]
        assert part["core"].tolist() == core
        sub = Adense[np.ix_(core, core)]                    # induced subgraph, brute force
        for i in range(len(core)):
            nb = part["col"][part["rowptr"][i]:part["rowptr"][i + 1]].tolist()
            assert nb == np.nonzero(sub[i])[0].tolist()
        assert part["d_g"].tolist() == Adense[core].sum(1).tolist()
        assert np.all(part["d_l"] <= part["d_g"]) and np.all(part["d_l"] >= 0)
        assert part["seeds"].tolist() == [i for i, v in enumerate(core) if train[v]]
        # symmetry of the local CSR
        L = np.zeros((len(core),) * 2, dtype=int)
        for i in range(len(core)):
            L[i, part["col"][part["rowptr"][i]:part["rowptr"][i + 1]]] = 1
        assert np.array_equal(L, L.T)


def test_full_coverage_and_chunk_pair_identity():
    wl = gen.small_workload("products", n=3000, scale=12, num_samples=30000)
    rp, col = gen.rmat(wl.scale, wl.n, wl.num_samples, 11, 12)
    # C=2: one pair covers the whole graph -> d_l = d_g
    ch2 = P.make_chunks(wl.n, 2, 5)
    full = P.induced_partition(rp, col, ch2, 0, 1)
    assert np.array_equal(full["d_l"], full["d_g"]) and full["core"].size == wl.n
    # exact chunk-pair identity from the C x C chunk edge-count matrix
    C = 5
    ch = P.make_chunks(wl.n, C, 6)
    row_of = np.repeat(np.arange(wl.n), np.diff(rp))
    E = np.zeros((C, C), dtype=np.int64)
    np.add.at(E, (ch[row_of], ch[col]), 1)
    for b, s in itertools.permutations(range(C), 2):
        part = P.induced_partition(rp, col, ch, b, s)
        assert part["col"].size == E[b, b] + E[s, s] + E[b, s] + E[s, b]


@pytest.mark.parametrize("C,W", [(4, 4), (5, 2), (3, 1)])
def test_one_cycle_covers_every_edge(C, W):
    n = 200
    rp, col = gen.rmat(8, n, 1500, 3, 4)
    ch = P.make_chunks(n, C, 8)
    seen = set()
    for row in P.sweep_schedule(C, W):
        for b, s in row:
            part = P.induced_partition(rp, col, ch, b, s)
            core = part["core"]
            for i in range(core.size):
                for j in part["col"][part["rowptr"][i]:part["rowptr"][i + 1]]:
                    seen.add((int(core[i]), int(core[j])))
    row_of = np.repeat(np.arange(n), np.diff(rp))
    assert seen == set(zip(row_of.tolist(), col.tolist()))


def test_base_equals_swept_rejected():
    rp, col = gen.csr_from_edges(3, [(0, 1)])
    with pytest.raises(ValueError):
        P.induced_partition(rp, col, np.array([0, 1, 1]), 1, 1)


def test_triangle_halo1_hand_example():
    g = GOLD["triangle_partition_halo1"]
    rp, col = gen.csr_from_edges(g["n"], g["edges"])
    part = P.induced_partition(rp, col, np.array(g["chunk_of"]), g["base"], g["swept"], halo=True)
    nc = part["n_core"]
    assert part["core"][:nc].tolist() == g["core"] and part["core"][nc:].tolist() == g["halo"]
    assert part["d_l"][:nc].tolist() == g["d_l_core"] and part["d_l"][nc:].tolist() == g["d_l_halo"]
    # node 0's row: global neighbours 1 (core, local 1) and 2 (halo, local 2), ascending gid
    assert part["col"][part["rowptr"][0]:part["rowptr"][1]].tolist() == [1, 2]


@pytest.mark.parametrize("seed", range(6))
def test_halo1_partition_brute_force(seed):
    """halo = {u not in core : some core v has u in N(v)}, by enumeration over the dense
    adjacency; core rows keep every neighbour (d_l = d_g), halo rows are empty, every local edge
    has a core endpoint, core and halo are disjoint, local ids core-then-halo ascending."""
    n = 29
    edges = _random_graph(n, 0.12, seed)
    rp, col = gen.csr_from_edges(n, edges)
    C = 5
    ch = P.make_chunks(n, C, seed + 7)
    train = (np.arange(n) % 2 == 0).astype(np.uint8)
    Adense = np.zeros((n, n), dtype=int)
    for u, v in edges:
        Adense[u, v] = Adense[v, u] = 1
    for b, s in itertools.permutations(range(C), 2):
        part = P.induced_partition(rp, col, ch, b, s, train, halo=True)
        core = [v for v in range(n) if ch[v] in (b, s)]
        halo = [u for u in range(n) if u not in core and any(Adense[v, u] for v in core)]
        nodes = core + halo
        assert part["n_core"] == len(core) and part["core"].tolist() == nodes
        for i, v in enumerate(nodes):
            nb = part["col"][part["rowptr"][i]:part["rowptr"][i + 1]].tolist()
            if i < len(core):
                assert [nodes[j] for j in nb] == np.nonzero(Adense[v])[0].tolist()
            else:
                assert nb == []
        assert part["d_l"][:len(core)].tolist() == part["d_g"][:len(core)].tolist()
        assert part["d_g"].tolist() == Adense[nodes].sum(1).tolist()
        assert part["seeds"].tolist() == [i for i, v in enumerate(core) if train[v]]
    # C = 2: one pair holds every node, no halo, identical to induced-core
    ch2 = P.make_chunks(n, 2, seed)
    a = P.induced_partition(rp, col, ch2, 0, 1, train, halo=True)
    b = P.induced_partition(rp, col, ch2, 0, 1, train)
    for k in ("core", "rowptr", "col", "d_l", "d_g", "seeds"):
        assert np.array_equal(a[k], b[k])
