"""Repartition (a3) probe on the products-shaped graph: one super-epoch switch = the 8 partitions
of sweep step t extracted from the replicated global CSR (bf16 features).  Prints per-switch wall
time (host, includes the syncs), the summed profiling-scope time and algorithmic GB/s.
Usage: python scripts/repart_probe.py [switches] [config]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402
from paper_2602_01872_b200.engine import sweep_schedule  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    name = sys.argv[2] if len(sys.argv) > 2 else "products"
    G.load()
    wl = gen.WORKLOADS[name]
    ds = gen.make_dataset(wl)
    ctx = G.Context(0)
    d = "cuda"
    rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
    x = torch.from_numpy(ds.x).to(torch.bfloat16).to(d)
    tr_, y = torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d)
    del ds
    C = wl.chunks
    ch = torch.empty(wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, wl.n, C, gen.seed_of("chunks"), ch)
    sched = sweep_schedule(C, C)
    index = G.Index(ctx, rp, col, ch, C)          # built once per run, as the engine does
    parts = [None] * C
    batch = hasattr(G, "grappa_repartition_batch") and os.environ.get("GRAPPA_PROBE_BATCH", "1") == "1"
    for r in range(reps + 1):
        pairs = sched[r % len(sched)]
        ctx.profile(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if batch:
            parts = G.grappa_repartition_batch(ctx, rp, col, x, "bf16", ch, C, pairs, tr_, y, parts, index=index)
        else:
            for w, (b, s) in enumerate(pairs):
                parts[w] = G.grappa_repartition(ctx, rp, col, x, "bf16", ch, C, b, s, tr_, y, parts[w])
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        ms, calls, by, _ = ctx.profile_read("repart")
        ctx.profile(False)
        if r > 0:
            print(f"switch {r} ({'batched' if batch else 'per partition'}): wall {wall:.2f} ms, "
                  f"scopes {ms:.2f} ms over {calls} calls, {by / 1e9:.3f} GB algorithmic, "
                  f"{by / (wall / 1e3) / 1e9:.0f} GB/s of wall", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
