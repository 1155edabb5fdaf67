"""Host/device trace of the mini-batch iteration (diagnostic): per-iteration wall time of
grappa_sample / grappa_minibatch_step / aggregate, then per-kernel-class device time.
Usage: python scripts/mb_trace.py [papers|small] [iters]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402
from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "small"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
if which == "papers":
    wl = gen.WORKLOADS["papers"]
else:
    wl = gen.small_workload("papers", n=20_000_000, scale=25, num_samples=300_000_000)
t = time.time()
ds = gen.make_dataset(wl)
print("gen", round(time.time() - t, 1), "s  nnz", ds.nnz, flush=True)
ctx = G.Context(0)
for kv in filter(None, os.environ.get("GRAPPA_VARIANTS", "").split(",")):   # e.g. tnrows=2,wstream=2
    k, v = kv.split("=")
    ctx.set_variant(k, int(v))
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
t = time.time()
tr = MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 8, gen.seed_of("chunks"),
                      fanouts=(15, 10, 5), batch_size=1000, sample_seed=5, dtype="bf16")
del ds
tr.repartition(1)
torch.cuda.synchronize()
print("trainer+repartition", round(time.time() - t, 1), "s", flush=True)
p = tr.parts[0]
print("part 0: n_core", p.n_core, "nnz", p.nnz, "seeds", p.n_seeds, flush=True)
order = torch.empty(p.n_seeds, dtype=torch.int32, device="cuda")
G.grappa_epoch_seeds(ctx, p, 5, 0, order)
torch.cuda.synchronize()
for it in range(5):
    t0 = time.perf_counter()
    seeds = order[it * 1000:(it + 1) * 1000]
    b = G.grappa_sample(ctx, p, seeds, [15, 10, 5], 5, 0, it, tr.batch, views=False)
    tr.batch = b
    t1 = time.perf_counter()
    need = G.minibatch_ws_bytes(b, spec.dims_pad, "bf16")
    if tr.mb_ws is None or tr.mb_ws.numel() < need:
        tr.mb_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    G.grappa_minibatch_step(ctx, p, b, spec.dims_pad, wl.K, tr.theta, tr.grad, tr.mb_ws, tr.loss_dev, "bf16")
    t2 = time.perf_counter()
    G.grappa_aggregate_grads_c(ctx, b.factors["resampling"], tr.grad, 1, 0.003, tr.theta)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"it {it}: sample {1e3*(t1-t0):.2f} ms  step-launch {1e3*(t2-t1):.2f} ms  agg+sync {1e3*(t3-t2):.2f} ms",
          flush=True)
ctx.profile(True)
t0 = time.perf_counter()
for it in range(5, 5 + iters):
    seeds = order[it * 1000:(it + 1) * 1000]
    b = G.grappa_sample(ctx, p, seeds, [15, 10, 5], 5, 0, it, tr.batch, views=False)
    tr.batch = b
    need = G.minibatch_ws_bytes(b, spec.dims_pad, "bf16")
    if tr.mb_ws.numel() < need:
        tr.mb_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    G.grappa_minibatch_step(ctx, p, b, spec.dims_pad, wl.K, tr.theta, tr.grad, tr.mb_ws, tr.loss_dev, "bf16")
    G.grappa_aggregate_grads_c(ctx, b.factors["resampling"], tr.grad, 1, 0.003, tr.theta)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"{iters} iterations: {1e3*wall/iters:.2f} ms/iteration wall", flush=True)
for k in ("sample", "spmm", "gemm", "gemm_tn", "loss", "agg"):
    ms, n, by, fl = ctx.profile_read(k)
    print(f"{k:8s} {ms/iters:8.3f} ms/iter  calls {n}", flush=True)
bi = b.refresh(3).blocks
print("last batch blocks:", [(x["n_dst"], x["n_src"], x["nnz"]) for x in bi], flush=True)
