"""CPU oracle for the sparse-sampler hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithms
(`/root/reference/pkg/src/sparse_sampler/{rng,density,estimators,pyramid,images,tonemap,losses}.py`,
and the score- and loss-gradient lines of `optimize.py`)
generalised to any odd kernel size k and any level count L.  It exists to
*check* the CUDA product path, never to stand in for it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2602_08642_b200`` never imports it (a test
  enforces this), and fails loudly when its CUDA library is missing.

Parity pin: at k = 5 the restatement reproduces the unmodified reference
bit-for-bit in float64 (tests/test_oracle_golden.py, against fixtures generated
by ``tests/golden/make_golden.py`` from the reference itself).
"""

from . import rng, density, estimators, pyramid, scores, temporal, tonemap  # noqa: F401
