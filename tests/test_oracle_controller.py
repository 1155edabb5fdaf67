"""Pins for the oracle's training controller (§3.5; reading R32) and
parity of the product-side controller (paper_2602_01872_b200.controller, pure host logic) with
it -- CPU only.

Pins: SPEC's hand examples (e = 100, C = 5 -> 25 epochs per super-epoch; fixed partitions never
switch; zero deficit switches only on the target length), the EMA written out by hand for a
short stream, and the streak rule at its threshold."""
import numpy as np
import pytest

from oracle.controller import Controller


def test_target_length_spec_example():
    c = Controller(epochs_total=100, num_chunks=5)            # target_length = 25
    assert c.target == 25
    decisions = []
    for _ in range(60):
        c.observe(1.0)                                          # full coverage: no deficit
        decisions.append(c.end_epoch())
    assert [i for i, d in enumerate(decisions) if d] == [24, 49]


def test_fixed_partitions_never_switch():
    c = Controller(epochs_total=10, num_chunks=3, fixed=True)   # S:463 (ablation FP)
    for _ in range(50):
        for _ in range(5):
            c.observe(0.0)
        assert not c.end_epoch()


def test_ema_by_hand():
    c = Controller(epochs_total=100, num_chunks=2, decay=0.9)
    xs = [0.2, 0.6, 0.4]
    for x in xs:
        c.observe(x)
    hand = 0.9 * (0.9 * 0.2 + 0.1 * 0.6) + 0.1 * 0.4
    assert abs(c.c_hat - hand) < 1e-15
    assert abs(c.deficit - (1 - hand)) < 1e-15


def test_deficit_streak_triggers_early_switch():
    c = Controller(epochs_total=1000, num_chunks=2, streak_threshold=20)   # target 1000
    # 19 steps of deficit 0.8 (> 0.5): no switch yet at the epoch boundary
    for _ in range(19):
        c.observe(0.2)
    assert c.streak == 19 and not c.end_epoch()
    c.observe(0.2)
    assert c.streak == 20 and c.end_epoch()                    # persisted -> early switch
    assert c.epochs_in == 0 and c.streak == 0 and c.c_hat is None
    # a single good step breaks the streak only once the EMA is back under the threshold
    for _ in range(25):
        c.observe(0.2)
    c2 = Controller(epochs_total=1000, num_chunks=2)
    for _ in range(25):
        c2.observe(0.2)
    c2.observe(1.0)                                            # EMA 0.28 -> deficit still > 0.5
    assert c2.streak == 26


def test_product_controller_matches_oracle():
    from paper_2602_01872_b200.controller import Controller as P
    rng = np.random.default_rng(0)
    for trial in range(20):
        e, C = int(rng.integers(5, 80)), int(rng.integers(2, 9))
        kw = dict(decay=float(rng.uniform(0.5, 0.99)), deficit_threshold=float(rng.uniform(0.1, 0.9)),
                  streak_threshold=int(rng.integers(1, 30)))
        a, b = Controller(e, C, **kw), P(e, C, **kw)
        for epoch in range(60):
            for _ in range(int(rng.integers(1, 9))):
                x = float(rng.uniform(0, 1)) if rng.random() < 0.7 else float(rng.uniform(0, 1e-6))
                a.observe(x)
                b.observe(x)
            assert a.end_epoch() == b.end_epoch(), (trial, epoch)
            assert a.streak == b.streak and a.epochs_in == b.epochs_in
