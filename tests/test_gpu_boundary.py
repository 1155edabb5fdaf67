"""The a7 boundary call's contract (include/grappa.h grappa_aggregate_grads), on the GPU:

* the coverage factor from the caller's eps / c_max (SPEC CorrectionConfig S:311-314, guards
  S:351 / S:383, reading R12) against oracle.correction.c_resampling with the same arguments;
* comm_dtype = bf16: the aggregated gradient is c/M * g rounded to bf16 once (the fused scale/cast
  before the all-reduce);
* a non-finite aggregated gradient never reaches theta ("non-finite grad -> error"): the
  device skips the SGD step and grappa_check reports E_NONFINITE;
* library-owned memory comes from the caller allocator (PyTorch's caching allocator) when the ctx
  is created with one, and results do not depend on the allocator;
* single-GPU training moves no cross-GPU bytes (grappa_comm_bytes)."""
import math

import numpy as np
import pytest
import torch

import gen
from oracle import correction as Co
from oracle import partition as Po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


@pytest.fixture(scope="module")
def ds():
    wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3)
    return gen.make_dataset(wl)


def _part(G, ctx, ds, C=8, b=2, s=5):
    d = "cuda"
    ch = torch.empty(ds.wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, ds.wl.n, C, gen.seed_of("chunks"), ch)
    return G.grappa_repartition(ctx, torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d),
                                torch.from_numpy(ds.x).to(d), "f32", ch, C, b, s,
                                torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d))


def _oracle_stats(ds, C=8, b=2, s=5):
    chunk_of = Po.make_chunks(ds.wl.n, C, gen.seed_of("chunks"))
    ref = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train)
    return ref["d_l"][ref["seeds"]], ref["d_g"][ref["seeds"]]


@pytest.mark.parametrize("eps,c_max", [(1e-9, 10.0), (1e30, 10.0), (1e-9, 1.0), (0.5, 2.0)])
def test_resampling_factor_uses_caller_guards(G, ds, eps, c_max):
    ctx = G.Context(0)
    part = _part(G, ctx, ds)
    s_dl, s_dg = _oracle_stats(ds)
    c_ref = Co.c_resampling(s_dl, s_dg, eps=eps, c_max=c_max)
    g = torch.linspace(-1, 1, 4096, device="cuda")
    grad = g.clone()
    G.grappa_aggregate_grads(ctx, part, "resampling", grad, 1, 0.0, None, eps=eps, c_max=c_max)
    torch.cuda.synchronize()
    ctx.check()
    ref = (g.double().cpu().numpy() * np.float32(c_ref)).astype(np.float32)
    assert np.array_equal(grad.cpu().numpy(), ref)           # one fp32 multiply: exact
    if eps > 1.0:
        assert c_ref == 1.0
    for bad in [dict(eps=0.0), dict(c_max=0.5)]:
        with pytest.raises(G.GrappaError, match="E_ARG"):
            G.grappa_aggregate_grads(ctx, part, "resampling", grad, 1, 0.0, None, **bad)
    ctx.close()


def test_comm_dtype_bf16(G, ds):
    ctx = G.Context(0)
    part = _part(G, ctx, ds)
    n = 117_120
    g = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    theta0 = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    for m, lr in [(1, 0.0), (2, 0.003)]:
        grad, theta = g.clone(), theta0.clone()
        G.grappa_aggregate_grads(ctx, part, "uniform", grad, m, lr, theta, comm_dtype="bf16")
        torch.cuda.synchronize()
        ctx.check()
        c = part.info.c_uniform
        want = (g * np.float32(c / m)).to(torch.bfloat16).float()
        assert torch.equal(grad, want)
        if lr:
            # the kernel's step is one FMA: theta - lr * g rounded once
            ref = (theta0.double() - float(np.float32(lr)) * want.double()).float()
            assert torch.allclose(theta, ref, rtol=2 ** -23, atol=0)
        # the same call with fp32 payload differs (the cast is real) but only by bf16 rounding
        g32 = g.clone()
        G.grappa_aggregate_grads(ctx, part, "uniform", g32, m, 0.0, None)
        torch.cuda.synchronize()
        assert not torch.equal(g32, grad)
        assert float((g32 - grad).abs().max() / g32.abs().max()) <= 2 ** -8
    with pytest.raises(G.GrappaError, match="E_ARG"):
        G.grappa_aggregate_grads(ctx, part, "uniform", g.clone(), 1, 0.0, None, comm_dtype=7)
    ctx.close()


@pytest.mark.parametrize("comm", ["f32", "bf16"])
def test_nonfinite_gradient_never_reaches_theta(G, ds, comm):
    ctx = G.Context(0)
    part = _part(G, ctx, ds)
    n = 50_000
    theta = torch.ones(n, device="cuda")
    grad = torch.full((n,), 0.5, device="cuda")
    grad[n // 2] = float("nan")
    G.grappa_aggregate_grads(ctx, part, "none", grad, 1, 0.1, theta, comm_dtype=comm)
    torch.cuda.synchronize()
    assert torch.equal(theta, torch.ones(n, device="cuda"))        # no partial update either
    with pytest.raises(G.GrappaError, match="E_NONFINITE"):
        ctx.check()
    # the flag is cleared by the check: the next finite step updates theta
    grad = torch.full((n,), 0.5, device="cuda")
    G.grappa_aggregate_grads(ctx, part, "none", grad, 1, 0.1, theta, comm_dtype=comm)
    torch.cuda.synchronize()
    ctx.check()
    assert torch.allclose(theta, torch.full((n,), 1.0 - 0.1 * 0.5, device="cuda"))
    # an overflow produced by the scale itself is caught the same way
    theta0 = theta.clone()
    grad = torch.full((n,), 3e38, device="cuda")
    G.grappa_aggregate_grads_c(ctx, 4.0, grad, 1, 0.1, theta, comm_dtype=comm)
    torch.cuda.synchronize()
    assert torch.equal(theta, theta0)
    with pytest.raises(G.GrappaError, match="E_NONFINITE"):
        ctx.check()
    ctx.close()


def test_caller_allocator_matches_cudamalloc(G, ds):
    """the same partition built through PyTorch's caching allocator and through cudaMalloc"""
    parts = []
    for torch_alloc in (True, False):
        ctx = G.Context(0, torch_alloc=torch_alloc)
        before = torch.cuda.memory_allocated()
        p = _part(G, ctx, ds)
        torch.cuda.synchronize()
        grown = torch.cuda.memory_allocated() - before
        parts.append((ctx, p, grown))
    (c1, p1, grown1), (c2, p2, grown2) = parts
    assert grown1 > 0                 # library buffers came from the torch pool
    for name in ("rowptr", "col", "core_global", "d_l", "d_g", "seeds", "x"):
        assert torch.equal(getattr(p1, name), getattr(p2, name)), name
    assert p1.info.c_resampling == p2.info.c_resampling
    # the partition outlives its ctx and is still freed through the allocator that made it
    c1.close()
    p1.destroy()
    c2.close()


def test_single_gpu_training_moves_no_cross_gpu_bytes(G, ds):
    from paper_2602_01872_b200.engine import ModelSpec, Trainer
    wl = ds.wl
    ctx = G.Context(0)
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, ModelSpec(wl.arch, wl.dims, wl.dims_pad),
                 ds.weights, wl.chunks, gen.seed_of("chunks"), repartition_every=1, dtype="bf16")
    tr.run_epoch()
    tr.run_epoch()
    torch.cuda.synchronize()
    tr.check()
    assert ctx.comm_bytes() == (0, 0)
    ctx.close()
    assert math.isfinite(float(tr.theta.sum()))
