"""Oracle: the training controller's switching rule (§3.5; SPEC S:406-409, S:456-464,
S:494-495).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:354: "a target of e/(c-1) super-epochs where e is a fixed number of epochs ... The controller
monitors a simple coverage deficit statistic per partition, Delta_t = 1 - c_hat_t, and triggers an
earlier repartition when Delta_t persists across several steps".  Reading R32 (DESIGN.md §2,
following SPEC S:459/S:494-495 where the paper gives no values):
  * target length L = ceil(e / (C - 1)) epochs per super-epoch (one sweep cycle over e epochs);
  * c_hat_t = exponential moving average of the per-iteration coverage factor (decay 0.9), started
    at the first observation of the super-epoch; one observation per optimizer step = the mean
    of the active partitions' factors in that phase-iteration (Alg. 1);
  * Delta_t = 1 - c_hat_t; streak = consecutive steps with Delta_t > 0.5;
  * at an epoch boundary: switch iff epochs_in_super_epoch >= L, or streak >= 20;
    fixed partitions (ablation FP) never switch;
  * a switch resets epochs_in_super_epoch, the EMA and the streak.
"""
from __future__ import annotations

import math


class Controller:
    def __init__(self, epochs_total: int, num_chunks: int, decay: float = 0.9,
                 deficit_threshold: float = 0.5, streak_threshold: int = 20, fixed: bool = False):
        if num_chunks < 2:
            raise ValueError("C >= 2")
        self.target = math.ceil(epochs_total / (num_chunks - 1))
        self.decay = decay
        self.deficit_threshold = deficit_threshold
        self.streak_threshold = streak_threshold
        self.fixed = fixed
        self.reset()

    def reset(self):
        self.epochs_in = 0
        self.c_hat = None
        self.streak = 0

    @property
    def deficit(self) -> float:
        return 0.0 if self.c_hat is None else 1.0 - self.c_hat

    def observe(self, c: float):
        """one optimizer step with (mean active) coverage factor c"""
        self.c_hat = c if self.c_hat is None else self.decay * self.c_hat + (1.0 - self.decay) * c
        self.streak = self.streak + 1 if self.deficit > self.deficit_threshold else 0

    def end_epoch(self) -> bool:
        """epoch boundary: True = repartition before the next epoch (and reset)"""
        self.epochs_in += 1
        if self.fixed:
            return False
        switch = self.epochs_in >= self.target or self.streak >= self.streak_threshold
        if switch:
            self.reset()
        return switch
