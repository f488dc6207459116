"""CPU oracle for the NS right-hand-side + RK hot path -- TEST INFRASTRUCTURE ONLY.

This package is the *checker*.  It restates, in numpy/scipy, the algorithm of
the reference package ``spectralrk`` (arxiv/paper_1810_10197) for the path the
B200 build accelerates: 3/2-rule dealiased pseudo-spectral Navier-Stokes /
Boussinesq tendencies, the RK4 / BS5 (DP5, KCL5) stage combinations, the
embedded-error norm, the step-size controller and the stepping loops.

Rules ("Oracle"):

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
  / ``--impl reference`` leg may import anything from here.  The product
  package ``paper_1810_10197_b200`` never does: its compute path is the CUDA
  library and it raises when that library is missing.
* The restatement is pinned against golden vectors produced by running the
  reference itself in the build container (``oracle/make_golden.py`` ->
  ``tests/golden/``), see ``tests/test_oracle_golden.py``.
* The FFT arithmetic of the reference lives in third-party libraries that are
  not vendored in ``/root/reference``: numpy.fft (pocketfft; numpy 2.3.5 here)
  and scipy.fft (ducc backend; scipy 1.18.1 here).  The oracle calls the same
  library entry points at the same call sites (``spectral.py:258-292``) so the
  restatement reproduces the reference bit for bit in this environment.
"""

from .spectral_np import *  # noqa: F401,F403
