"""CPU oracle for the batched keyed-hash path (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It is the checker, never
the product: the engine in ``paper_1612_06257_b200`` has no CPU fallback.

``lh_oracle.c`` restates the reference ``lanehash`` algorithm (file:line
citations in its header); it is pinned against the reference's frozen
vectors and reference-generated fixtures by tests/test_oracle.py.
"""
