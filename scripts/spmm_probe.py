"""SpMM kernel probe on a products-shaped partition (bf16, GCN hidden layer 128 -> 128): times
the aggregation per kernel variant with the library's profiling scopes (CUDA events).
Usage: python scripts/spmm_probe.py [reps] [variants, e.g. 0,2] [width] [flags]
flags: grappa_layer_fwd_ex flags, e.g. 8 = GCN input layer (aggregate-first: the weighted
gather over the source norms at width f_in), 4 = node-level (weighted by d_l/d_g)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    variants = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,2").split(",")]
    width = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    G.load()
    wl = gen.WORKLOADS["products"]
    ds = gen.make_dataset(wl)
    ctx = G.Context(0)
    d = "cuda"
    ch = torch.empty(wl.n, dtype=torch.int32, device=d)
    G.grappa_partition(ctx, wl.n, 8, gen.seed_of("chunks"), ch)
    x = torch.from_numpy(ds.x).to(torch.bfloat16).to(d)
    part = G.grappa_repartition(ctx, torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d), x, "bf16",
                                ch, 8, 0, 1, torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d))
    n = part.n_core
    print(f"partition: n={n} nnz={part.nnz} n_heavy={part.info.n_heavy} n_slots={part.info.n_slots}", flush=True)
    g = torch.Generator(device=d).manual_seed(1)
    h = torch.randn(n, width, device=d, generator=g).to(torch.bfloat16)
    w = (torch.randn(width, width, device=d, generator=g) / 11).contiguous()
    out = torch.empty(n, width, device=d, dtype=torch.bfloat16)
    ws = torch.empty(G.layer_ws_bytes(part, "gcn", width, width, "bf16") * 2, dtype=torch.uint8, device=d)
    saved = torch.empty(max(1, G.layer_saved_bytes(part, "gcn", width, width, "bf16", flags)), dtype=torch.uint8,
                        device=d)
    ref = None
    for v in variants:
        ctx.set_variant("spmm", v)
        for _ in range(2):
            G.grappa_layer_fwd_ex(ctx, part, "gcn", width, width, True, h, w, out, saved, ws, "bf16", flags)
        torch.cuda.synchronize()
        ctx.profile(True)
        for _ in range(reps):
            G.grappa_layer_fwd_ex(ctx, part, "gcn", width, width, True, h, w, out, saved, ws, "bf16", flags)
        ms, calls, by, _ = ctx.profile_read("spmm")
        ctx.profile(False)
        torch.cuda.synchronize()
        same = None
        if ref is None:
            ref = out.clone()
        else:
            same = torch.equal(out.view(torch.int16), ref.view(torch.int16))
            if not same:
                e = ((out.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
                same = f"False (max rel diff {e:.2e})"
        print(f"variant {v}: spmm {ms / calls * 1e3:.1f} us/call, {by / calls / 1e9:.3f} GB algorithmic, "
              f"{by / (ms / 1e3) / 1e9:.0f} GB/s, bitwise == first variant: {same}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
