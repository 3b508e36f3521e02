"""TEST INFRASTRUCTURE — the parity oracle for the reference's hot path.

Two restatements of pairsim's gate-sweep / measure path
(/root/reference/pkg/src/pairsim/kernel.py:31-165, measure.py:29-99):

* ``oracle.c``   — ctypes binding of qsim_oracle.c (liboracle.so), scalar C
  with the exact numpy FMA arithmetic; the bit-exact checker.
* ``oracle.port`` — a numpy port of the reference's vectorised sweep with its
  ThreadExecutor chunking; the CPU baseline that bench.py times.

Both are pinned against the reference itself by tests/test_oracle.py using
the golden vectors in tests/golden/ (generated from pairsim by
tests/golden/make_golden.py).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg may import this package;
the product (paper_1805_00988_b200) never does.
"""
