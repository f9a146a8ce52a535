"""CPU oracle for the DAE-subspace Newton-step hot path (TEST INFRASTRUCTURE ONLY).

This package is a numpy-fp64 restatement of the reference algorithm of
arXiv 2102.11026 as specified in /root/reference/SPEC.md, built on a
restatement of the reference multicomplex kernels (pkg/src/nlrom/mcx.py).
It is the checker, never the thing measured or shipped: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product path (``paper_2102_11026_b200`` / ``nlrom``) never imports it.

Parity pinning
--------------
* ``oracle.mcx_np`` (multicomplex part kernels) is PINNED: it is checked
  against golden vectors produced by the reference ``nlrom/mcx.py`` itself
  (``tests/golden/make_golden.py`` → ``tests/golden/mcx_golden.npz``) and
  against re-derivations of every check in the reference test file
  ``pkg/tests/test_mcx.py`` (closed forms, Taylor ring oracle, complex128,
  CR homomorphism).
* The decoder CSFD bundle is pinned to the reference arithmetic by golden
  vectors computed with the reference ``mcx`` part kernels on small nets
  (``tests/golden/decoder_golden.npz``).
* Everything above (elastic StVK, cubature, rdsim assembly / Newton step)
  has no reference code (SPEC only). It is pinned by the SPEC known-answer
  tests (Fig. 5 values 36/18, hvv=18, svv=24, f_fict=4, dJ=24, ...) and by
  the SPEC's own brute-force oracles (per-entry CSFD, jacobian_oracle =
  CSFD of the residual). Parity at that boundary is therefore "pinned by
  SPEC KATs + CSFD oracles, not by reference outputs".
"""
