"""Timing probe of the split-fp32 transform GEMM (diagnostic): GCN layer forward at products
partition shape (n = 612k, 128 -> 128, fp32), GEMM class time per call with the x3dbg knob
(1 = no A loads, 2 = no output stores, 4 = no weight staging, 8 = hi*hi MMA only,
16 = no epilogue work); results are invalid for dbg != 0."""
import sys, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa
import paper_2602_01872_b200 as G  # noqa
wl = gen.WORKLOADS["products"]
ds = gen.make_dataset(wl)
ctx = G.Context(0)
d = "cuda"
rp, col = torch.from_numpy(ds.rowptr).to(d), torch.from_numpy(ds.col).to(d)
ch = torch.empty(wl.n, dtype=torch.int32, device=d)
G.grappa_partition(ctx, wl.n, 8, gen.seed_of("chunks"), ch)
part = G.grappa_repartition(ctx, rp, col, torch.from_numpy(ds.x).to(d), "f32", ch, 8, 0, 1,
                            torch.from_numpy(ds.train).to(d), torch.from_numpy(ds.y).to(d))
n = part.n_core
lib = G.load()
import sys as _s
dts = _s.argv[1:] or ["f32", "bf16"]
for dt, fi, fo, arch in [(t, 128, 128, a) for t in dts for a in ("gcn", "sage")]:
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    h = torch.randn(n, fi, device=d).relu().to(tdt)
    w = torch.randn((2 if arch == "sage" else 1) * fi, fo, device=d) / 10
    out = torch.empty(n, fo, device=d, dtype=tdt)
    saved = torch.empty(max(1, G.layer_saved_bytes(part, arch, fi, fo, dt)), dtype=torch.uint8, device=d)
    ws = torch.empty(G.layer_ws_bytes(part, arch, fi, fo, dt), dtype=torch.uint8, device=d)
    for dbg in ((0, 4, 7, 100) if dt == "f32" else (0, 100)):
        if dbg == 100:
            lib.grappa_set_kernel_variant(b"gemm", 1)
            lib.grappa_set_kernel_variant(b"x3dbg", 0)
        else:
            lib.grappa_set_kernel_variant(b"x3dbg", dbg)
        for _ in range(2):
            G.grappa_layer_fwd(ctx, part, arch, fi, fo, True, h, w, out, saved, ws, dt)
        torch.cuda.synchronize()
        ctx.profile(True)
        for _ in range(10):
            G.grappa_layer_fwd(ctx, part, arch, fi, fo, True, h, w, out, saved, ws, dt)
        torch.cuda.synchronize()
        ms, calls, byts, fl = ctx.profile_read("gemm")
        ctx.profile(False)
        print(f"{dt} {arch} n={n} {fi}->{fo} dbg={dbg}: {ms / calls * 1e3:.1f} us/call, {byts / (ms / 1e3) / 1e9:.0f} GB/s")
    lib.grappa_set_kernel_variant(b"gemm", 0)
    lib.grappa_set_kernel_variant(b"x3dbg", 0)
