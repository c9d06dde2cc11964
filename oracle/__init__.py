"""CPU oracle for the SU(3) hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the arithmetic of the reference package
``su3bench`` (arXiv 1309.0551, /root/reference/pkg/src/su3bench) for the eight
routines on the hot path and the lattice sweeps composed from them.  It is the
checker the CUDA path is compared against; it is never the thing measured or
shipped.

Who may import it (and nobody else):
  * ``tests/``                      -- parity tests;
  * ``__graft_entry__.smoke()``     -- one tiny check on cuda:0;
  * ``bench.py``                    -- the ``cpu_baseline`` leg and ``--impl reference``.

The product package ``paper_1309_0551_b200`` does not import this package and
fails loudly when its CUDA library is missing; there is no CPU fallback.

Pinning: ``routines`` and ``sweeps`` are checked bit-for-bit against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``); the C restatement
``su3_oracle.c`` is checked bit-for-bit against the numpy restatement.
"""
