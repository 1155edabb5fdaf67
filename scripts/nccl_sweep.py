"""All-reduce bandwidth through the product path: grappa_aggregate_grads_c --
the fused c_p/M scale + non-finite flag kernel followed by ncclAllReduce(sum) on the flat fp32
gradient -- timed with CUDA events on the launching stream, max over ranks, for buffer sizes from
1 KB to 1 GB and at the real gradient sizes of the configs (205-737 KB).
  algbw = bytes / time,  busbw = algbw * 2 (G - 1) / G   (compare with 900 GB/s per direction)
Needs >= 2 GPUs (one process per GPU):
  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 scripts/nccl_sweep.py
With one process there is no collective to time (the call is the scale kernel only) and the
script says so."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01872_b200 as G  # noqa: E402

# flat parameter counts of the configs' models: cora, arxiv, products, papers, R-MAT
REAL = {"cora": 184_320, "arxiv": 75_776, "products": 117_120, "papers": 109_568, "rmat": 51_200}


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:
        print(json.dumps({"all_reduce": "not timed: one process (grappa_aggregate_grads_c issues no "
                                        "collective when nranks = 1); launch with torchrun on >= 2 GPUs"}))
        return
    dist.init_process_group("nccl", device_id=dev)
    uid = G.Context.nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0)
    ctx = G.Context(local, rank, world, bytes(t.cpu().tolist()))
    stream = torch.cuda.current_stream(dev)
    sizes = sorted({1 << k for k in range(10, 31, 2)} | {4 * n for n in REAL.values()})
    rows = []
    for nbytes in sizes:
        n = max(1, nbytes // 4)
        g = torch.ones(n, dtype=torch.float32, device=dev)
        reps = 50 if nbytes <= (8 << 20) else 10
        for _ in range(5):
            G.grappa_aggregate_grads_c(ctx, 1.0, g, world, 0.0, None, stream)
        dist.barrier()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            G.grappa_aggregate_grads_c(ctx, 1.0, g, world, 0.0, None, stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        sec = float(ms.item()) / 1e3
        alg = 4 * n / sec / 1e9
        rows.append({"bytes": 4 * n, "us": sec * 1e6, "algbw_GBps": alg,
                     "busbw_GBps": alg * 2 * (world - 1) / world,
                     "config": next((k for k, v in REAL.items() if 4 * v == 4 * n), None)})
    ctx.check(stream)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "peak_GBps_per_direction": 900, "rows": rows}))
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
