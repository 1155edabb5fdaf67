# host-overhead trace of the papers mini-batch iteration (diagnostic)
import time, sys, torch
sys.path.insert(0, "/root/repo")
import gen
import paper_2602_01872_b200 as G
from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec
wl = gen.small_workload("papers", n=20_000_000, scale=25, num_samples=300_000_000)
t=time.time(); ds = gen.make_dataset(wl); print("gen", time.time()-t, ds.nnz, flush=True)
ctx = G.Context(0)
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
tr = MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 8, gen.seed_of("chunks"),
                      fanouts=(15,10,5), batch_size=1000, sample_seed=5, dtype="bf16")
tr.repartition(1)
p = tr.parts[0]
order = torch.empty(p.n_seeds, dtype=torch.int32, device="cuda")
G.grappa_epoch_seeds(ctx, p, 5, 0, order)
nb = tr.iterations(p)
torch.cuda.synchronize()
for it in range(5):
    t0 = time.perf_counter()
    seeds = order[it*1000:(it+1)*1000]
    b = G.grappa_sample(ctx, p, seeds, [15,10,5], 5, 0, it, tr.batch, views=False); tr.batch = b
    t1 = time.perf_counter()
    need = G.minibatch_ws_bytes(b, spec.dims_pad, "bf16")
    if tr.mb_ws is None or tr.mb_ws.numel() < need: tr.mb_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    G.grappa_minibatch_step(ctx, p, b, spec.dims_pad, wl.K, tr.theta, tr.grad, tr.mb_ws, tr.loss_dev, "bf16")
    t2 = time.perf_counter()
    G.grappa_aggregate_grads_c(ctx, b.factors["resampling"], tr.grad, 1, 0.003, tr.theta)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"it {it}: sample {1e3*(t1-t0):.2f} ms  step-launch {1e3*(t2-t1):.2f} ms  agg+sync {1e3*(t3-t2):.2f} ms", flush=True)
ctx.profile(True)
for it in range(5, 25):
    seeds = order[it*1000:(it+1)*1000]
    b = G.grappa_sample(ctx, p, seeds, [15,10,5], 5, 0, it, tr.batch, views=False); tr.batch = b
    need = G.minibatch_ws_bytes(b, spec.dims_pad, "bf16")
    if tr.mb_ws.numel() < need: tr.mb_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    G.grappa_minibatch_step(ctx, p, b, spec.dims_pad, wl.K, tr.theta, tr.grad, tr.mb_ws, tr.loss_dev, "bf16")
torch.cuda.synchronize()
for k in ("sample","spmm","gemm","gemm_tn","loss"):
    print(k, ctx.profile_read(k))
