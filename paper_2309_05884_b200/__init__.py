"""B200-native GRAPE fidelity+gradient engine (arXiv 2309.05884 hot path).

Host side (Python, mirrors the reference ``symqoc`` API): Pauli operators,
D_n / S_n block bases, the BASELINE systems, ``qoc.gradient`` /
``objective(u) -> (F, grad)`` and the optimiser drivers.  Device side:
hand-written sm_100a kernels behind the C ABI in ``include/symqoc_b200.h``.
"""

__version__ = "0.1.0"
