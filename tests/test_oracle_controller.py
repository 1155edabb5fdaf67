"""Pins for the oracle's training controller (§3.5; reading R32) and
parity of the product-side controller (paper_2602_01872_b200.controller, pure host logic) with
it -- CPU only.

Pins: SPEC's hand examples (e = 100, C = 5 -> 25 epochs per super-epoch; fixed partitions never
switch; zero deficit switches only on the target length), the EMA written out by hand for a
short stream, per partition, the default deficit threshold relative to a random chunk pair's
coverage 2/C, the streak rule at its threshold, and the lowest-coverage partition deciding."""
import numpy as np
import pytest

from oracle.controller import Controller


def test_target_length_spec_example():
    c = Controller(epochs_total=100, num_chunks=5)            # target_length = 25
    assert c.target == 25
    decisions = []
    for _ in range(60):
        c.observe(0, 1.0)                                       # full coverage: no deficit
        decisions.append(c.end_epoch())
    assert [i for i, d in enumerate(decisions) if d] == [24, 49]


def test_fixed_partitions_never_switch():
    c = Controller(epochs_total=10, num_chunks=3, fixed=True)   # S:463 (ablation FP)
    for _ in range(50):
        for p in range(5):
            c.observe(p, 0.0)
        assert not c.end_epoch()


def test_ema_by_hand_per_partition():
    c = Controller(epochs_total=100, num_chunks=2, decay=0.9)
    xs = [0.2, 0.6, 0.4]
    for x in xs:
        c.observe(3, x)
        c.observe(5, 1.0 - x)                                   # another partition's own EMA
    hand = 0.9 * (0.9 * 0.2 + 0.1 * 0.6) + 0.1 * 0.4
    assert abs(c.c_hat[3] - hand) < 1e-15
    assert abs(c.deficit(3) - (1 - hand)) < 1e-15
    assert abs(c.c_hat[5] - (0.9 * (0.9 * 0.8 + 0.1 * 0.4) + 0.1 * 0.6)) < 1e-15


def test_default_threshold_is_relative_to_random_pair_coverage():
    """R32: threshold 1 - (1/2)(2/C).  Random chunking gives a chunk pair coverage 2/C in
    expectation, so a partition AT that coverage never fires (C = 8: coverage 0.25, deficit 0.75
    < 0.875), one at a third of it does after streak_threshold steps"""
    for C in (2, 4, 8):
        c = Controller(epochs_total=10_000, num_chunks=C)
        assert abs(c.deficit_threshold - (1 - 1 / C)) < 1e-15
        for _ in range(200):
            c.observe(0, 2.0 / C)
        assert c.streak[0] == 0 and not c.end_epoch()
        c = Controller(epochs_total=10_000, num_chunks=C, streak_threshold=20)
        for k in range(19):
            c.observe(0, 2.0 / (3 * C))
        assert not c.end_epoch()
        c.observe(0, 2.0 / (3 * C))
        assert c.end_epoch()


def test_deficit_streak_triggers_early_switch():
    c = Controller(epochs_total=1000, num_chunks=2, deficit_threshold=0.5, streak_threshold=20)
    # 19 steps of deficit 0.8 (> 0.5): no switch yet at the epoch boundary
    for _ in range(19):
        c.observe(0, 0.2)
    assert c.streak[0] == 19 and not c.end_epoch()
    c.observe(0, 0.2)
    assert c.streak[0] == 20 and c.end_epoch()                 # persisted -> early switch
    assert c.epochs_in == 0 and c.streak == {} and c.c_hat == {}
    c2 = Controller(epochs_total=1000, num_chunks=2, deficit_threshold=0.5)
    for _ in range(25):
        c2.observe(0, 0.2)
    c2.observe(0, 1.0)                                         # EMA 0.28 -> deficit still > 0.5
    assert c2.streak[0] == 26


def test_lowest_coverage_partition_decides():
    """P:356 "prioritizing partitions with low coverage": one partition with a persistent deficit
    switches the super-epoch although the others are well covered; interleaving does not reset
    its streak"""
    c = Controller(epochs_total=1000, num_chunks=4, streak_threshold=5)
    for k in range(5):
        for p in range(4):
            c.observe(p, 0.9 if p != 2 else 0.01)
        assert c.end_epoch() == (k == 4)
    assert c.c_hat == {}


def test_product_controller_matches_oracle():
    from paper_2602_01872_b200.controller import Controller as P
    rng = np.random.default_rng(0)
    for trial in range(20):
        e, C = int(rng.integers(5, 80)), int(rng.integers(2, 9))
        kw = dict(decay=float(rng.uniform(0.5, 0.99)), streak_threshold=int(rng.integers(1, 30)))
        if trial % 2:
            kw["deficit_threshold"] = float(rng.uniform(0.1, 0.9))
        a, b = Controller(e, C, **kw), P(e, C, **kw)
        for epoch in range(60):
            for _ in range(int(rng.integers(1, 9))):
                p = int(rng.integers(0, C))
                x = float(rng.uniform(0, 1)) if rng.random() < 0.7 else float(rng.uniform(0, 1e-6))
                a.observe(p, x)
                b.observe(p, x)
            assert a.end_epoch() == b.end_epoch(), (trial, epoch)
            assert a.streak == b.streak and a.epochs_in == b.epochs_in
