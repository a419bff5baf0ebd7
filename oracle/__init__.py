"""CPU oracle for the ReCoGS recolor hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference `splattint`
algorithm (``/root/reference/pkg/src/splattint``), written from the
reference's documented semantics; every function cites the reference
``file:line`` it follows.  It exists to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2511_18441_b200`` never imports it and has no
  CPU fallback -- it fails loudly when its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
the real reference (``tests/golden/make_golden.py`` imports ``splattint`` from
``/root/reference`` in the build container and writes ``tests/golden/*.npz``)
and against the known-answer cases of the reference's own tests
(pkg/tests/test_render.py, test_selection.py, test_losses.py, ...), see
``tests/test_oracle_golden.py``.  The exact-decision arithmetic (the
world->camera FMA chain that numpy/OpenBLAS uses for ``P @ R.T + t``) is also
restated in plain C in ``oracle/c/rcgs_oracle.c`` and checked against numpy on
whichever host runs the tests.
"""

from .config import (  # noqa: F401
    ALPHA_CLAMP, ALPHA_SKIP, COV_DILATION, FOOTPRINT_SIGMAS, NEAR_CLIP, T_FLOOR,
    DEPTH_TAU, SSIM_C1, SSIM_C2, LAMBDA,
)
