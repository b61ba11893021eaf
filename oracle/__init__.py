"""CPU oracle for the FusedLoRA / FusedMultiLoRA hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or the timed
CPU baseline. The product (``paper_2510_00206_b200``) never imports it and has no CPU
fallback.

Contents (each module cites the reference lines it restates):
  philox.py   Philox4x32-10 (Random123) + SPEC.md §3 keep mask, vectorised numpy
  lora.py     Eq. 1 forward/backward at SPEC.md §2's rounding points, fp64 accumulation
  routing.py  segment table -> 16 B / 128-row routing table (ls/costmodel.py:23-26, 279-281)
  traffic.py  independent byte-count restatement of ls/costmodel.py:219-306 (+ b200_minimal)

Pinning status:
  * traffic bytes — pinned to the reference: tests/golden/traffic_reference.json is produced
    by importing lorasched.costmodel itself (tests/golden/make_reference_golden.py) and the
    frozen totals of pkg/tests/test_costmodel.py:22-27.
  * Philox — pinned to the published Random123 known-answer vectors (tests/test_oracle.py).
  * routing / segments — pinned to lorasched's own packing semantics (padded_len, segment
    order) through tests/golden/schedule_reference.json, a schedule planned by lorasched
    itself (tests/golden/make_reference_golden.py).
  * DP balance — tests/golden/c5_simulate_dp.json, lorasched.pipesim.simulate_dp on the C5
    bench's rank streams (tests/golden/make_dp_golden.py).
  * Y, dX, dA, dB numerics — PARITY UNPINNED by the reference: lorasched has no numerical
    implementation of the path (SPEC.md:8 of the reference puts the kernels out of scope).
    The oracle restates Eq. 1 and is cross-checked against an
    independent torch-CPU float64 autograd restatement of the same equations.
"""
