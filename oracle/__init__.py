"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow CPU implementation of what the hot path computes, written from
PAPER.md (arXiv 2307.12059) and pinned by tests/test_oracle_*.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import, call, link or execute anything here.
The product package (paper_2307_12059_b200/) never imports it and shares no
code with it; the CUDA path fails loudly when its extension is missing.

Parity status per function:
  join / dist3 / dist_rows     pinned (hand examples, scipy cdist, brute force, invariants)
  pivot_distances              pinned (closed forms, Lemma 1 property)
  compute_range                pinned (SPEC worked example, Eq. (11) brute force)
  group_candidates             pinned (paper's grouping example)
  calibrate_theta / compare    harness helpers (not method arithmetic)
"""
