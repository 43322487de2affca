"""CPU oracle for the GRAPE fidelity+gradient hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
as the timed CPU reference -- never as the product path.  The product path
(``paper_2309_05884_b200``) runs the sm_100a kernels and fails loudly when the
CUDA library is missing.

Pinning: ``tests/golden/*.npz`` hold outputs of the reference package itself
(``/root/reference/pkg/src/symqoc``, run in the build container by
``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks this oracle
against them.
"""
