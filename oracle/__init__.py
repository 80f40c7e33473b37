"""CPU oracle for the decode-time MoE offloading path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference package
``moe_offload`` (``/root/reference/pkg/src/moe_offload``) for the hot path the
B200 engine replaces: group quantization (``quant.py``), the decode model math
(``model.py``), the two-tier LRU/staging expert store (``store.py``) and the
session / offload / replay flow (``engine.py``).  Every function cites the
reference ``file:line`` it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import it, and only as the *checker* or the
timed CPU baseline.  The product package ``paper_2312_17238_b200`` never
imports this package and has no CPU fallback.

Parity pinning: the restatement is checked against golden vectors produced by
the unmodified reference (``tests/golden/make_golden.py``) and against the
reference's own known-answer tests (2-bit checksum 0.36625814, bits/param
2.640625, the LRU golden sequence, gate KATs).
"""
