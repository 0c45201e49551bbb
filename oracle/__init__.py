"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the ApplyFilter / Fill path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the reference-arm
timing.  The product path (``paper_2203_10213_b200``) never imports it.
See ``oracle/vkt_oracle.py`` for the restatement and its pinning.
"""
