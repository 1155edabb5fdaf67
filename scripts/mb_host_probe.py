"""Is the pipelined mini-batch epoch host-bound?  (diagnostic)  Runs MinibatchTrainer epochs on a
papers-shaped graph and splits the host wall time into time blocked in grappa_sample_wait (the host
waiting for a batch's block sizes) and the rest (issuing launches); GPU epoch time by CUDA events.
Usage: python scripts/mb_host_probe.py [papers|small] [depth]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402
import paper_2602_01872_b200 as pkg  # noqa: E402
from paper_2602_01872_b200.engine import MinibatchTrainer, ModelSpec  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "small"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = gen.WORKLOADS["papers"] if which == "papers" else gen.small_workload(
    "papers", n=20_000_000, scale=25, num_samples=300_000_000)
ds = gen.make_dataset(wl)
ctx = G.Context(0)
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
tr = MinibatchTrainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, 8, gen.seed_of("chunks"),
                      fanouts=(15, 10, 5), batch_size=1000, sample_seed=5, dtype="bf16", depth=depth)
del ds
blocked = [0.0]
orig = pkg.grappa_sample_wait


def timed_wait(b, views=True):
    t = time.perf_counter()
    r = orig(b, views)
    blocked[0] += time.perf_counter() - t
    return r


pkg.grappa_sample_wait = timed_wait
tr.run_epoch()                       # warm (repartition, allocations)
torch.cuda.synchronize()
for _ in range(2):
    blocked[0] = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    tr.run_epoch()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"epoch: gpu {e0.elapsed_time(e1):.1f} ms, host wall {1e3 * wall:.1f} ms, blocked in sample_wait "
          f"{1e3 * blocked[0]:.1f} ms, host busy {1e3 * (wall - blocked[0]):.1f} ms", flush=True)
