"""Training controller: when to leave the current super-epoch (§3.5; reading R32 in
DESIGN.md, the SPEC S:459/S:494-495 defaults).

Host control only (no GPU work).  Rule: after an epoch, repartition iff the super-epoch has
lasted ceil(e / (C - 1)) epochs, or the coverage deficit 1 - EMA_0.9(c) has exceeded 0.5 for the
last 20 optimizer steps; a fixed-partition run (ablation FP) never repartitions.  The observed c
of a step is the mean factor of the phase's active partitions; multi-rank runs feed every rank
the same sequence (Trainer gathers the per-step factors once per epoch), so every rank takes the
same decision without a per-step collective.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Controller:
    epochs_total: int
    num_chunks: int
    decay: float = 0.9
    deficit_threshold: float = 0.5
    streak_threshold: int = 20
    fixed: bool = False
    epochs_in: int = field(default=0, init=False)
    streak: int = field(default=0, init=False)
    c_hat: float | None = field(default=None, init=False)

    def __post_init__(self):
        if self.num_chunks < 2:
            raise ValueError("controller needs C >= 2 chunks")
        q, r = divmod(self.epochs_total, self.num_chunks - 1)
        self.target = q + (1 if r else 0)

    def observe(self, c: float) -> None:
        prev = self.c_hat
        self.c_hat = c if prev is None else prev * self.decay + c * (1.0 - self.decay)
        if 1.0 - self.c_hat > self.deficit_threshold:
            self.streak += 1
        else:
            self.streak = 0

    def end_epoch(self) -> bool:
        self.epochs_in += 1
        go = (not self.fixed) and (self.epochs_in >= self.target or self.streak >= self.streak_threshold)
        if go:
            self.epochs_in, self.streak, self.c_hat = 0, 0, None
        return go
