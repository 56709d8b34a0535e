"""StragglAR oracle — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU reference for the
StragglAR straggler-aware AllReduce (arXiv 2505.23523, /root/reference/PAPER.md).
It exists to *check* the CUDA path, never to serve it:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it.
* It shares no code with ``paper_2505_23523_b200`` (the product package) and
  never imports it.  The only module both sides use is the seeded input
  generator ``paper_2505_23523_b200/inputs.py``, which holds none of the
  method's arithmetic.

Citations use ``P:<line>`` for PAPER.md and ``S:<line>`` for SPEC.md, followed
by the section / algorithm / equation the line falls in.

Modules
-------
schedule   Algorithm 1 schedule generator, Appendix B matcher,
           Ring / RHD / Broadcast baseline schedules, contributor-set
           verifier, per-round invariants of App. A.
numerics   Plain definition of the AllReduce result, Phase A (ReduceScatter among
           non-stragglers) and the snapshot replay of Phase B, direct
           completion, ring-order / butterfly (RHD) / Broadcast oracles, bf16
           round-to-nearest-even, tolerance of SURVEY.md §8(c).6.
cost       alpha-beta closed forms of Table 1, T_RS, critical delay
           (P:423-424).

Parity status: every public function here is pinned by a ``-m "not gpu"``
test in ``tests/test_oracle_*.py`` (DESIGN.md §8 lists each with its pin); the
private helpers (``_canonical_partial``, ``log2_exact``, ``generate``,
``replay_schedule``, ``initial_state_*``) are exercised only through the pinned
functions that call them, and DESIGN.md §8 names those.  Helpers that no pin
covered (a holder-set trace and a JSON exporter) were removed in round 2 rather
than left "parity unpinned".
"""
