"""Training controller: when to leave the current super-epoch (§3.5; reading R32 in
DESIGN.md, the SPEC S:459/S:494-495 defaults).

Host control only (no GPU work).  Rule: after an epoch, repartition iff the super-epoch has
lasted ceil(e / (C - 1)) epochs, or some partition's coverage deficit 1 - EMA_0.9(coverage) has
exceeded the threshold (default 1 - 1/C: below half the 2/C coverage random chunking gives a
chunk pair) for its last 20 optimizer steps -- the lowest-coverage partition decides (P:356
"prioritizing partitions with low coverage"); a fixed-partition run (ablation FP) never
repartitions.  The coverage of a step is the partition's mean d_l/d_g over its seeds (the
eq:correction_uniform average), independent of the correction applied to the gradient.
Multi-rank runs feed every rank the same (partition, coverage) sequence (Trainer gathers the
per-step records once per epoch), so every rank takes the same decision without a per-step
collective.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Controller:
    epochs_total: int
    num_chunks: int
    decay: float = 0.9
    deficit_threshold: float | None = None
    streak_threshold: int = 20
    fixed: bool = False
    epochs_in: int = field(default=0, init=False)
    c_hat: dict = field(default_factory=dict, init=False)
    streak: dict = field(default_factory=dict, init=False)

    def __post_init__(self):
        if self.num_chunks < 2:
            raise ValueError("controller needs C >= 2 chunks")
        q, r = divmod(self.epochs_total, self.num_chunks - 1)
        self.target = q + (1 if r else 0)
        if self.deficit_threshold is None:
            self.deficit_threshold = 1.0 - 1.0 / self.num_chunks

    def observe(self, part: int, c: float) -> None:
        prev = self.c_hat.get(part)
        ema = c if prev is None else prev * self.decay + c * (1.0 - self.decay)
        self.c_hat[part] = ema
        self.streak[part] = self.streak.get(part, 0) + 1 if 1.0 - ema > self.deficit_threshold else 0

    def end_epoch(self) -> bool:
        self.epochs_in += 1
        worst = max(self.streak.values()) if self.streak else 0
        go = (not self.fixed) and (self.epochs_in >= self.target or worst >= self.streak_threshold)
        if go:
            self.epochs_in, self.c_hat, self.streak = 0, {}, {}
        return go
