"""Debug: GAT on halo-1 partitions -- compare the trainer's hidden activations of phase 0 with
the oracle's forward (no borrowed masks), split into core and halo rows."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import gen
from oracle import model as Mo, partition as Po
import paper_2602_01872_b200 as G
from paper_2602_01872_b200.engine import ModelSpec, Trainer

G.load()
ctx = G.Context(0)
wl = gen.small_workload("products", n=20011, scale=15, num_samples=540_000, depth=3, arch="gat")
ds = gen.make_dataset(wl)
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
for halo in (False, True):
    tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
                 gen.seed_of("chunks"), corr="uniform", lr=0.05, repartition_every=1, dtype="f32", halo=halo)
    snaps = []
    def grab():
        if snaps: return
        p = tr.parts[0]
        snaps.append([tr.H[l][:p.n_core, :wl.dims[l]].float().cpu().numpy().astype(np.float64) for l in range(1, wl.depth)])
        snaps.append((p.n_core, p.n_halo))
    tr.run_epoch(on_phase=grab)
    torch.cuda.synchronize()
    P = wl.chunks
    chunk_of = Po.make_chunks(wl.n, P, gen.seed_of("chunks"))
    b, s = Po.sweep_schedule(P, P)[0][0]
    part = Po.induced_partition(ds.rowptr, ds.col, chunk_of, b, s, ds.train, halo=halo)
    X = ds.x[:, :wl.F].astype(np.float64)
    W0 = [[np.asarray(ws[0], np.float64)[:wl.dims[l], :wl.dims[l + 1]],
           np.asarray(ws[1], np.float64)[:2, :wl.dims[l + 1]]] for l, ws in enumerate(ds.weights)]
    _, g, _, cache = Mo.partition_loss_grad("gat", part, X[part["core"]], ds.y[part["core"]], W0, None)
    n_core, n_halo = snaps[1]
    print("halo", halo, "gpu n_core(local)", n_core, "n_halo", n_halo, "oracle rows", len(part["core"]),
          "oracle keys", list(part.keys()))
    for l in range(wl.depth - 1):
        Z = np.asarray(cache["Z"][l]); Hg = snaps[0][l]
        Ho = np.maximum(Z, 0)
        print(" layer", l + 1, "shapes", Z.shape, Hg.shape)
        m = min(len(Ho), len(Hg))
        d = np.abs(Hg[:m] - Ho[:m]).max(1) / max(np.abs(Ho).max(), 1e-30)
        nc = n_core - n_halo
        print("   core rows err max", d[:nc].max() if nc else None, "bad", int((d[:nc] > 1e-4).sum()),
              " halo rows err max", d[nc:].max() if m > nc else None, "bad", int((d[nc:] > 1e-4).sum()))
        bad = np.nonzero(d > 1e-4)[0][:10]
        print("   first bad rows", bad)
ctx.close()
