"""CPU oracle for the explicit wave-stepping hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithms of `wavecell`
(arXiv 2501.19013) that the B200 product replaces:

* ``oracle.timeint`` -- numpy/scipy restatement of ``cdm_run``,
  ``imex_run``, ``newmark_run``, ``max_gen_eig`` (src/timeint.py,
  src/linalg.py).  SciPy's CSR matvec and SuperLU are the same third-party
  arithmetic the reference calls (scipy >= 1.10, pkg/pyproject.toml:10-13;
  1.18.1 in this image).
* ``wc_oracle.c`` -- a C restatement of the CSR CDM loop and CSR assembly of
  structured spectral-cell operators, used as the multi-threaded CPU baseline
  (``bench.py --impl reference`` / ``cpu_baseline``) on the GPU box, where
  the Python reference does not exist.
* ``oracle.geometry_cube`` -- the reference's rotated-cube benchmark
  geometry (src/geometry.py:128-272), which pins the product's host set-up
  to the reference's own grids and operators.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the reference itself in this container
(``tests/golden/make_golden.py``; fixtures in ``tests/golden/*.npz``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package -- as the checker, never as the thing measured
or shipped.  The product (``paper_2501_19013_b200``) never imports it.
"""
