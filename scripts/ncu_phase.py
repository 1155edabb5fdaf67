"""Profiler window of exactly one Alg. 1 phase of the bench workload (diagnostic, for ncu).

Builds the same Trainer bench.py times, runs one warm epoch, then brackets ONE phase
(fwd / loss / bwd / aggregate of partition 0) with cudaProfilerStart/Stop, so that
  ncu --profile-from-start off --set full ... python scripts/ncu_phase.py
captures every kernel of that phase once.  The number of LOGICAL calls per kernel class
(one SpMM call = its degree-bucket launches + fix-up) is written next to the report so
scripts/ncu_summary.py can state DRAM traffic per logical call, the unit bench.py's
roofline `achieved` uses.
Usage: python scripts/ncu_phase.py [config] [dtype] [out.json]   (default gpurun_out/ncu_phase_calls.json)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2602_01872_b200 as G  # noqa: E402
from paper_2602_01872_b200 import _lib  # noqa: E402
from paper_2602_01872_b200.engine import ModelSpec, Trainer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "products"
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
wl = gen.WORKLOADS[cfg]
ds = gen.make_dataset(wl)
ctx = G.Context(0)
spec = ModelSpec(wl.arch, wl.dims, wl.dims_pad)
tr = Trainer(ctx, ds.rowptr, ds.col, ds.x, ds.y, ds.train, spec, ds.weights, wl.chunks,
             gen.seed_of("chunks"), corr=wl.correction, lr=0.003,
             repartition_every=wl.repartition_every, dtype=dtype,
             num_workers=wl.extra.get("workers"))
del ds
tr.run_epoch()
torch.cuda.synchronize()
ctx.profile(True)
i, w = tr.my_workers()[0]
torch.cuda.cudart().cudaProfilerStart()
tr.phase_step(i, w, 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
calls = {k: ctx.profile_read(k)[1] for k in _lib.KCLASS}
alg = {k: ctx.profile_read(k)[2] for k in _lib.KCLASS}
ctx.profile(False)
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "ncu_phase_calls.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
with open(out, "w") as f:
    json.dump({"config": cfg, "dtype": dtype, "worker": w, "logical_calls": calls,
               "algorithmic_bytes": alg}, f)
