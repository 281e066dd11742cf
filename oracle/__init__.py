"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the Uzawa hot path.

This package is a CPU restatement (numpy + scipy, the reference's own
third-party numerics) of the algorithm implemented by the reference package
``pintsolve`` (arXiv 1802.08126 reference, ``/root/reference/pkg``).  Every
function cites the reference ``file:line`` it restates.

It is the *checker*, never the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_1802_08126_b200`` never imports it and has no
  CPU fallback -- it fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle.py`` checks this restatement bit-for-bit against
golden vectors produced by the unmodified reference
(``tests/golden/make_golden.py``, run in the build container where the
reference is importable).
"""

from .pint_oracle import *  # noqa: F401,F403
