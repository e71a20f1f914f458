"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the CUDA path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package. The product package
(``paper_2501_19004_b200``) never imports it and has no CPU fallback.

Two checkers:

* ``oracle.port`` — plain-C restatement of the reference hot path
  (``oracle/lvn_oracle.c``, built to ``oracle/_build/liboracle.so``).
* ``oracle.ref`` — the unmodified reference library compiled from
  ``/root/reference/proj/core/src`` (``oracle/_ref/libref.so``) behind a C shim.

The restatement is pinned against the reference's own golden values
(``tests/golden``) and against ``oracle.ref`` (``tests/test_oracle_*.py``).
"""

from .oracle import (  # noqa: F401
    Csr,
    OracleError,
    build,
    port,
    ref,
    ref_available,
)
