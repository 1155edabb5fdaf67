"""Shared parity helpers for the GPU tests (test infrastructure, no method arithmetic).

err(x, y)   max|x - y| / max|y| -- the parity metric of SURVEY §8(c) c.4 (y = the f64 oracle).
TOL         the north_star bars: 1e-4 (fp32 storage), 2e-2 (bf16 storage).
FLIP        reading R16b: where a test evaluates the oracle with the ReLU decisions
            the kernels took (the masks the GPU's hidden activations imply), each decision may
            differ from the oracle's own 1[Z > 0] only at a pre-activation within rounding of 0:
            |Z| <= FLIP[dtype] * max|Z| of that layer (fp32: 1e-5; bf16: the bf16 bar itself,
            the size of the difference the kernels' Z may legitimately have).
assert_flips_bounded(cache, dtype)
            checks every layer of an oracle forward cache (oracle.model.forward /
            oracle.sampler.sage_forward: lists Z and M) against that bound; so no test feeds
            kernel-made decisions to the oracle unchecked.
"""
import numpy as np

TOL = {"f32": 1e-4, "bf16": 2e-2}
FLIP = {"f32": 1e-5, "bf16": 2e-2}


def err(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)) if y.size else 0.0


def assert_flips_bounded(cache, dtype, where=""):
    """R16b flip bound over every layer of an oracle forward cache; returns the flip count."""
    thr = FLIP[dtype]
    total = 0
    for l, (Z, M) in enumerate(zip(cache["Z"], cache["M"])):
        Z = np.asarray(Z, dtype=np.float64)
        flip = (Z > 0) != (np.asarray(M) > 0)
        nf = int(flip.sum())
        if nf:
            zmax = float(np.max(np.abs(Z)))
            worst = float(np.max(np.abs(Z[flip])))
            assert worst <= thr * zmax, (f"{where} layer {l}: {nf} ReLU decisions differ from the oracle's, "
                                         f"worst |Z| = {worst:.3e} > {thr} * max|Z| = {thr * zmax:.3e}")
        total += nf
    return total
