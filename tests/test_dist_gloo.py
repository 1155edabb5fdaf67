"""N > 1 host logic on CPU: world_size-2 `gloo` process groups run the engine's phase plan
(phase i -> worker i*G + rank, m_active per phase, idle ranks contribute zeros) with the
oracle's per-partition gradients and a real all-reduce, and must reproduce the oracle's
single-process Algorithm 1 with M = G.  The CUDA path's equivalent collective
is the ncclAllReduce inside grappa_aggregate_grads (exercised on a GPU box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
from oracle import correction as Co
from oracle import model as Mo
from oracle import partition as Po
from oracle import train as Tr
from paper_2602_01872_b200.engine import phase_plan


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(C):
    wl = gen.small_workload("products", n=1500, scale=11, num_samples=12_000, depth=2, chunks=C,
                            hidden=16)
    ds = gen.make_dataset(wl)
    W0 = [[np.asarray(w, np.float64)[:wl.dims[l], :wl.dims[l + 1]] for w in ws]
          for l, ws in enumerate(ds.weights)]
    return wl, ds, W0


def _worker(rank, world, port, C, corr, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, ds, W0 = _setup(C)
    chunk_of = Po.make_chunks(wl.n, C, gen.seed_of("chunks"))
    pairs = Po.sweep_schedule(C, C)[0]
    shapes = [[w.shape for w in ws] for ws in W0]
    theta = Mo.flatten(W0)
    X = ds.x[:, :wl.F].astype(np.float64)
    for i, w, m_active in phase_plan(C, world, rank):
        g = np.zeros_like(theta)
        c = 0.0
        if w is not None:
            part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, *pairs[w], ds.train)
            _, g, _, _ = Mo.partition_loss_grad(wl.arch, part, X[part["core"]], ds.y[part["core"]],
                                                Mo.unflatten(theta, shapes))
            c = Tr.partition_factor(corr, part)
        t = torch.from_numpy(c / m_active * g)          # fused scale before the all-reduce
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        theta = Co.sgd(theta, t.numpy(), 0.1)
    th = torch.from_numpy(theta)
    dist.broadcast(th0 := th.clone(), 0)
    if rank == 0:
        out.put(theta)
    assert np.array_equal(theta, th0.numpy())          # replicas stay identical
    dist.destroy_process_group()


@pytest.mark.parametrize("C,corr", [(4, "uniform"), (3, "none"), (4, "resampling")])
def test_two_rank_phase_loop_matches_oracle(C, corr):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, C, corr, q)) for r in range(2)]
    for p in procs:
        p.start()
    theta = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    wl, ds, W0 = _setup(C)
    chunk_of = Po.make_chunks(wl.n, C, gen.seed_of("chunks"))
    final, recs = Tr.run(wl.arch, ds.rowptr, ds.col, ds.x[:, :wl.F].astype(np.float64), ds.y,
                         ds.train, W0, chunk_of, C, C, 2, corr, 0.1, 1, 10)
    assert len(recs) == -(-C // 2)
    ref = Mo.flatten(final)
    assert np.max(np.abs(theta - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_phase_plan():
    assert phase_plan(8, 1, 0) == [(i, i, 1) for i in range(8)]
    assert phase_plan(8, 8, 3) == [(0, 3, 8)]
    assert phase_plan(8, 4, 1) == [(0, 1, 4), (1, 5, 4)]
    assert phase_plan(3, 2, 1) == [(0, 1, 2), (1, None, 1)]
    # every worker runs exactly once per epoch across ranks ("every partition
    # contributes exactly one update per epoch")
    for W in range(1, 9):
        for G in range(1, 9):
            ws = sorted(w for r in range(G) for _, w, _ in phase_plan(W, G, r) if w is not None)
            assert ws == list(range(W))


def _ctrl_worker(rank, world, port, out):
    """each rank sees different coverages (its own partitions); after gathering the per-step
    (partition, coverage, active) lists once per epoch (Trainer.end_epoch) every rank must take
    the same switch decisions, equal to the oracle controller fed every active partition's step"""
    from paper_2602_01872_b200.controller import Controller
    from paper_2602_01872_b200.engine import merge_step_factors
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    ctrl = Controller(30, 4, streak_threshold=5)
    decisions = []
    for epoch in range(25):
        steps = []
        for i, w, m in phase_plan(3, world, rank):     # W = 3: rank 1 idle in phase 1
            steps.append((float(w), float(rng.uniform(0.0, 0.35)), 1.0) if w is not None
                         else (0.0, 0.0, 0.0))
        mine = torch.tensor(steps, dtype=torch.float64).reshape(-1, 3)
        every = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(every, mine)
        lists = [e.tolist() for e in every]
        for p, c in merge_step_factors(lists):
            ctrl.observe(p, c)
        decisions.append(ctrl.end_epoch())
        out.put((rank, epoch, lists))
    out.put((rank, "decisions", decisions))
    dist.destroy_process_group()


def test_two_rank_controller_agrees():
    from oracle.controller import Controller as OC
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ctrl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    lists = {}
    for _ in range(2 * 26):
        r, k, v = q.get(timeout=300)
        if k == "decisions":
            got[r] = v
        elif r == 0:
            lists[k] = v
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert got[0] == got[1]
    oc = OC(30, 4, streak_threshold=5)
    ref = []
    for epoch in range(25):
        per_rank = lists[epoch]
        for k in range(len(per_rank[0])):
            for r in per_rank:
                if r[k][2] > 0:
                    oc.observe(int(r[k][0]), r[k][1])
        ref.append(oc.end_epoch())
    assert got[0] == ref and any(ref)


def test_shard_plan():
    """sharded mode (a3 (i)): every worker ends each phase holding both chunks of its pair; with
    W = C = G the plan is the shift permutation (rank r receives chunk (r+t) mod C from its owner)"""
    from paper_2602_01872_b200.engine import shard_owner, shard_plan, sweep_schedule
    for C in range(2, 9):
        for G in range(1, C + 1):
            for W in sorted({C, max(1, C - 1)}):
                for pairs in sweep_schedule(C, W):
                    plan = shard_plan(pairs, W, G)
                    assert len(plan) == -(-W // G)
                    for i, xs in enumerate(plan):
                        for r in range(G):
                            w = i * G + r
                            if w >= W:
                                continue
                            held = {c for c in range(C) if shard_owner(c, G) == r}
                            held |= {c for (c, src, dst) in xs if dst == r}
                            assert set(pairs[w]) <= held
                        assert all(src != dst and shard_owner(c, G) == src for c, src, dst in xs)
    for C in (2, 4, 8):
        for t, pairs in enumerate(sweep_schedule(C, C), start=1):
            (xs,) = shard_plan(pairs, C, C)
            assert sorted(xs) == sorted(((r + t) % C, (r + t) % C, r) for r in range(C))


def _shard_worker(rank, world, port, C, out):
    """the engine's per-phase transfer lists (shard_plan / shard_xfers) driven through real gloo
    point-to-point sends: every rank receives exactly the chunk rows its worker's pair needs"""
    from paper_2602_01872_b200.engine import shard_owner, shard_plan, shard_xfers, sweep_schedule
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, ds, _ = _setup(C)
    chunk_of = Po.make_chunks(wl.n, C, gen.seed_of("chunks"))

    def rows(c):        # a shard's ids and concatenated adjacency (host stand-in)
        ids = np.flatnonzero(chunk_of == c)
        return ids, np.concatenate([ds.col[ds.rowptr[v]:ds.rowptr[v + 1]] for v in ids])

    owned = {c: rows(c) for c in range(C) if shard_owner(c, world) == rank}
    ok = True
    for pairs in sweep_schedule(C, C):
        for i, xs in enumerate(shard_plan(pairs, C, world)):
            snd, rcv = shard_xfers(xs, rank)
            reqs = []
            for dst, c in snd:
                ids, col = owned[c]
                bufs = [torch.tensor([c, ids.size, col.size], dtype=torch.int64),
                        torch.from_numpy(ids.astype(np.int64)), torch.from_numpy(col.astype(np.int64))]
                reqs += [dist.isend(b, dst) for b in bufs]
            got = {}
            for src, c in rcv:
                hdr = torch.empty(3, dtype=torch.int64)
                dist.recv(hdr, src)
                ids = torch.empty(int(hdr[1]), dtype=torch.int64)
                col = torch.empty(int(hdr[2]), dtype=torch.int64)
                dist.recv(ids, src)
                dist.recv(col, src)
                got[int(hdr[0])] = (ids.numpy(), col.numpy())
                ok &= int(hdr[0]) == c
            for r in reqs:
                r.wait()
            w = i * world + rank
            if w < C:
                for c in pairs[w]:
                    have = owned.get(c) or got.get(c)
                    ref = rows(c)
                    ok &= have is not None and np.array_equal(have[0], ref[0]) and np.array_equal(have[1], ref[1])
            dist.barrier()
    out.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("C", [2, 4])
def test_two_rank_shard_exchange(C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, C, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


def _shared_worker(rank, world, port, root, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = gen.small_workload("products", n=3001, scale=12, num_samples=30_000, depth=2, chunks=4, hidden=16)
    ds = gen.shared_dataset(wl, rank, lambda: dist.barrier(), root=root)
    d = {k: np.array(getattr(ds, k)) for k in ("rowptr", "col", "x", "y", "train")}
    d["w"] = np.concatenate([np.asarray(w).ravel() for ws in ds.weights for w in ws])
    out[rank] = d
    dist.destroy_process_group()


def test_shared_dataset_two_ranks(tmp_path):
    """bench at N > 1: rank 0 generates the inputs once and the other ranks map its copy
    (gen.shared_dataset) -- every rank sees exactly the generator's arrays"""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shared_worker, args=(world, _port(), str(tmp_path), out), nprocs=world, join=True)
    wl = gen.small_workload("products", n=3001, scale=12, num_samples=30_000, depth=2, chunks=4, hidden=16)
    ref = gen.make_dataset(wl)
    for r in range(world):
        for k in ("rowptr", "col", "x", "y", "train"):
            assert np.array_equal(out[r][k], getattr(ref, k)), (r, k)
        assert np.array_equal(out[r]["w"], np.concatenate([np.asarray(w).ravel() for ws in ref.weights for w in ws]))
    assert any(p.name.endswith("_col.npy") for p in tmp_path.iterdir())
