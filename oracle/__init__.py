"""CPU oracle for the per-Newton-iteration hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `intact` package's hot
path (`/root/reference/pkg/src/intact/{distance,bvh,ccd,elasticity,contact,
sparse,solver,stepper}.py`).  Every function cites the reference file:line it
restates.  It exists to check the CUDA path, nothing else:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
  `--impl reference` legs may import it;
* the product package (`paper_2512_12151_b200`) never imports it and has no
  CPU fallback — it fails loudly when `libibf.so` is missing.

Parity pinning: the restatement is pinned against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`), checked by
`tests/test_oracle_golden.py`.  Distance / ACCD / broad-phase / active-set
outputs are pinned bit-exactly; LAPACK-backed quantities (SVD, eigh, inv,
roots) are pinned to the reference's own tolerances because numpy's LAPACK is
unpinned (`pyproject.toml:11` says numpy>=1.24, no lockfile).

Reduction orders that matter for bit-exactness were probed on the build host
(numpy 2.3.5, AVX-512): `einsum('...k,...k->...')` of 3 terms evaluates
`(a0*b0 + a2*b2) + a1*b1`; `norm(axis=-1)` is sequential; mean of 3 is
`((a+b)+c)/3`; `np.sum` of 12 is numpy's 8-accumulator pairwise sum.  The
oracle spells those orders out explicitly so that it does not depend on the
SIMD dispatch of whichever host runs it.
"""
