"""CPU oracle for the R²CCL data-parallel hot path (arXiv 2512.25059).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2512_25059_b200``) never imports it and
shares no code with it; the only common module is ``r2inputs`` (seeded input
generators, no arithmetic of the method).

Plain, slow, sequential Python + numpy, written from the paper and
the SURVEY.md §8(c) readings.  Citations use ``P:n`` = PAPER.md line n and
``S:n`` = SPEC.md line n.

Modules
-------
semantic       Layer 1: the allreduce result (ring fold order, per-hop rounding).
geometry       shards / channel slices / chunks / stream positions (§8 header).
ledger         DMA-buffer rollback and the failover chain.
balance        R²CCL-Balance proportional redistribution.
triangulation  emulated zero-byte probes + three-point triangulation.
protocol       Layer 2: sequential simulator of the whole fault-tolerant ring
               allreduce (a3-a11 of SURVEY §8(a)), seeded interleavings.
cost           traffic / time bounds (App. A).

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against
values the paper / SPEC print, closed forms, library routines or brute force.
No function is "parity unpinned" (DESIGN.md §4 lists each pin).
"""
