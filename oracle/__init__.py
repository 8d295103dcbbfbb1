"""CPU oracle for the L4 hot path (arxiv 2512.19179) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2512_19179_b200``) never imports it, and this package never
imports the product: the two share no code.  Inputs come from ``synth/``.

Modules
-------
attention  paged GQA decode attention, FP64, the plain definition
           (PAPER.md:94-101 decode over cached KV; PAPER.md:677 paged KV).
partition  the §4.2 DP stage partition (Eq. (1) at
           PAPER.md:301-315) step by step, plus an exhaustive enumerator.
pool       page allocator + KV-page migration semantics.

Pins: see tests/test_oracle_*.py and DESIGN.md §"Oracle and pins".
"""
