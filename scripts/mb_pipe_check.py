"""Diagnostic: one pipelined mini-batch epoch (MinibatchTrainer.run_epoch) over all 8 partitions
of a scaled-down papers graph, then the same epoch unpipelined from the same theta; the final
theta must agree bitwise (sampling is deterministic and the step order is unchanged)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402
from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
scale = max(4, (n - 1).bit_length())
wl = gen.small_workload("papers", n=n, scale=scale, num_samples=n * 15, train_frac=0.05)
ds = gen.make_dataset(wl)
ctx = G.Context(0)
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
mk = lambda: MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 8,
                              gen.seed_of("chunks"), fanouts=(15, 10, 5), batch_size=1000, sample_seed=5,
                              dtype="bf16", corr="uniform", lr=0.01)
a = mk()
a.run_epoch()
torch.cuda.synchronize()
ctx.check()
b = mk()
# unpipelined reference: same phases, one grappa_sample (sync) per batch
from paper_2602_01872_b200 import grappa_aggregate_grads_c, grappa_epoch_seeds  # noqa: E402
from paper_2602_01872_b200.engine import phase_plan  # noqa: E402
b.repartition(1)
for i, w, m in phase_plan(b.W, b.G, b.rank):
    part = b.parts[w]
    order = torch.empty(part.n_seeds, dtype=torch.int32, device="cuda")
    grappa_epoch_seeds(ctx, part, b.sample_seed, 0, order, b.stream)
    nb = b.iterations(part)
    for it in range(nb):
        bt = b.minibatch(part, order, it, nb)
        grappa_aggregate_grads_c(ctx, bt.factors["uniform"], b.grad, m, b.lr, b.theta, b.stream)
torch.cuda.synchronize()
ctx.check()
d = (a.theta - b.theta).abs().max().item()
print(f"n={n} parts={[p.n_core for p in a.parts.values()]} max|theta_pipe - theta_seq| = {d}")
assert d == 0.0
print("pipelined == sequential: OK")
