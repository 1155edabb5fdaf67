"""Oracle: the training controller's switching rule (§3.5; SPEC S:406-409, S:456-464,
S:494-495).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:354-356: "a target of e/(c-1) super-epochs where e is a fixed number of epochs ... The
controller monitors a simple coverage deficit statistic per partition, Delta_t = 1 - c_hat_t, and
triggers an earlier repartition when Delta_t persists across several steps, prioritizing
partitions with low coverage".  Reading R32 (SPEC S:459/S:494-495 where the paper
gives no values):
  * target length L = ceil(e / (C - 1)) epochs per super-epoch (one sweep cycle over e epochs);
  * c_hat is a COVERAGE statistic, kept per partition p: the EMA (decay 0.9, started at p's first
    step of the super-epoch) of p's coverage c_cov = mean over its seeds of d_l/d_g (the
    eq:correction_uniform average), whatever correction the gradient uses -- the
    literal resampling factor (~1e-7 at the configs) is not a coverage;
  * Delta_p = 1 - c_hat_p; the deficit threshold is relative to the coverage random chunking
    gives a chunk pair in expectation (a neighbour lands in one of the two chunks with
    probability 2/C): default threshold = 1 - kappa * 2/C with kappa = 1/2, i.e. fire only when a
    partition sees less than half the coverage its layout predicts (C = 8: Delta > 0.875);
  * streak_p = consecutive steps of partition p with Delta_p > threshold;
  * at an epoch boundary: switch iff epochs_in_super_epoch >= L, or the lowest-coverage
    partition's deficit has persisted, max_p streak_p >= 20 ("prioritizing partitions with low
    coverage": with the deterministic sweep every worker advances together, so the partition
    with the worst coverage decides for all); fixed partitions (ablation FP) never switch;
  * a switch resets epochs_in_super_epoch, every EMA and every streak.
"""
from __future__ import annotations

import math


class Controller:
    def __init__(self, epochs_total: int, num_chunks: int, decay: float = 0.9,
                 deficit_threshold: float | None = None, streak_threshold: int = 20,
                 fixed: bool = False):
        if num_chunks < 2:
            raise ValueError("C >= 2")
        self.target = math.ceil(epochs_total / (num_chunks - 1))
        self.decay = decay
        # default: 1 - (1/2)(2/C) = 1 - 1/C
        self.deficit_threshold = (1.0 - 1.0 / num_chunks) if deficit_threshold is None \
            else deficit_threshold
        self.streak_threshold = streak_threshold
        self.fixed = fixed
        self.reset()

    def reset(self):
        self.epochs_in = 0
        self.c_hat = {}          # partition -> EMA of its coverage
        self.streak = {}         # partition -> consecutive steps over the threshold

    def deficit(self, p) -> float:
        return 1.0 - self.c_hat[p] if p in self.c_hat else 0.0

    def observe(self, p, c: float):
        """one optimizer step of partition p with coverage c (mean d_l/d_g over its seeds)"""
        prev = self.c_hat.get(p)
        self.c_hat[p] = c if prev is None else self.decay * prev + (1.0 - self.decay) * c
        self.streak[p] = self.streak.get(p, 0) + 1 if self.deficit(p) > self.deficit_threshold else 0

    def end_epoch(self) -> bool:
        """epoch boundary: True = repartition before the next epoch (and reset)"""
        self.epochs_in += 1
        if self.fixed:
            return False
        worst = max(self.streak.values(), default=0)
        switch = self.epochs_in >= self.target or worst >= self.streak_threshold
        if switch:
            self.reset()
        return switch
