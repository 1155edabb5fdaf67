"""CPU oracle for Grappa's partition-isolated training step (arXiv 2602.01872).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
from here.  The product path (``paper_2602_01872_b200``) never imports, links or
executes this package, and this package never imports the product path; the two
share no code.  The only shared module is ``gen`` (seeded input generators, no
method arithmetic).

Plain, slow, obviously-correct NumPy/SciPy in float64, following PAPER.md step by
step (citations ``P:<line>`` are PAPER.md lines; ``S:<line>`` SPEC.md lines; the
readings where the paper is silent are DESIGN.md §2 "Readings" R1..R20).

Modules
  partition   a1/a2/a3: random chunking, sweep schedule, induced chunk-pair partition
  model       a4/a5/a6: GCN / GraphSAGE layer forward, softmax-CE loss, exact backward
  correction  a7/a8:    coverage factors c_uniform / c_resampling (+HM reading),
                        (1/M) sum_p c_p g_p aggregation, SGD
  train       a9:       Algorithm 1 phase loop with super-epoch repartitioning

Pins (tests/test_oracle_*.py) tie every function to something other than itself:
hand values printed in SPEC.md, closed forms, brute force on tiny graphs, a dense
adjacency-matrix re-derivation, central finite differences and Theorem 2's projection.
Parity status of each function is listed in DESIGN.md §5; none is "parity unpinned".
"""
