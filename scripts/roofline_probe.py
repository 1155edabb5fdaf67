"""Measured ceilings for the roofline report (grappa_roofline_probe): HBM copy, L2-resident
streaming read and L2-resident whole-row gather at several table sizes.  Prints one JSON object.
Usage: python scripts/roofline_probe.py [out.json]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_01872_b200 as G  # noqa: E402


def main():
    G.load()
    ctx = G.Context(0)
    MB = 1 << 20
    out = {"gpu": torch.cuda.get_device_name(0)}
    out["hbm_copy_GBps"] = max(ctx.roofline_probe("hbm_copy", 2048 * MB, iters=5) for _ in range(3))
    out["l2_read_GBps"] = {str(m): max(ctx.roofline_probe("l2_read", m * MB, iters=10) for _ in range(3))
                           for m in (16, 32, 64, 96)}
    out["l2_gather_GBps"] = {f"{rb}B@{m}MB": max(ctx.roofline_probe("l2_gather", m * MB, row_bytes=rb, iters=10)
                                                 for _ in range(3))
                             for rb in (256, 128, 64) for m in (16, 32, 64, 96, 160, 512)}
    try:
        out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks.mem",
                                            "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except Exception as e:  # pragma: no cover
        out["nvidia_smi"] = str(e)
    js = json.dumps(out, indent=1)
    print(js)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(js)
    ctx.close()


if __name__ == "__main__":
    main()
