"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithm of the greedy
lookahead-decoding hot path (reference: ``/root/reference/pkg/src/lookahead``,
cited per function as ``<file>:<line>``).  It exists to *check* the B200 path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import it;
* the product package ``paper_2402_02057_b200`` never imports it and has no
  CPU fallback -- it fails loudly when the CUDA library is missing.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``oracle/make_golden.py`` -> ``tests/golden/``) plus the reference test-suite's
own known answers.
"""
