"""Golden vectors for the Trotterised per-qubit propagator, from the REFERENCE itself.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_trotter_golden.py

Writes tests/golden/r02_trotter.npz with outputs of symqoc.trotter (trotter.py:48-225):

* expm_2x2 on seeded Hermitian 2 x 2 matrices;
* PerQubitPlan.apply_step on a seeded state (n = 5) and step_unitary (n = 4), plain and Strang,
  one and two coupling offsets;
* fidelity_replay traces: n = 3 (40 steps, every step), n = 4 Strang (200 steps), n = 5 with two
  offsets at tau = 0.1, n = 6 (500 steps), the acceptance criterion-8 configuration
  (test_acceptance.py:212-226: ModelConfig(n, 1.0, (0.2,), "per-qubit"), tau = 0.05, 20000 steps)
  at n = 3..6 recorded every 100 steps, and n = 8 over 2000 steps;
* the error-order slope inputs of test_trotter.py:103-113 (n = 3: tau = 0.1, 0.05, 0.025 to T = 25).
"""

from __future__ import annotations

import os
import time

import numpy as np
from symqoc import model, trotter

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "r02_trotter.npz")


def main():
    z = {}
    rng = np.random.default_rng(2024)
    hs = []
    for _ in range(8):
        a = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        hs.append(a + a.conj().T)
    z["expm_h"] = np.array(hs)
    z["expm_tau"] = np.array([0.05, 0.3, 1.0, 2.0, 0.01, 0.7, 0.2, 1.5])
    z["expm_out"] = np.array([trotter.expm_2x2(h, t) for h, t in zip(hs, z["expm_tau"])])

    for tag, n, cpl in (("a", 5, (0.2,)), ("b", 5, (0.2, 0.1))):
        cfg = model.ModelConfig(n, 1.0, cpl, "per-qubit")
        psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        psi /= np.linalg.norm(psi)
        bx = rng.uniform(-1, 1, n)
        by = rng.uniform(-1, 1, n)
        z[f"step_{tag}_psi"], z[f"step_{tag}_bx"], z[f"step_{tag}_by"] = psi, bx, by
        for strang in (False, True):
            plan = trotter.PerQubitPlan(cfg, 0.05, strang=strang)
            z[f"step_{tag}_out_{int(strang)}"] = plan.apply_step(psi, bx, by)
    cfg4 = model.ModelConfig(4, 1.0, (0.2,), "per-qubit")
    bx, by = trotter.benchmark_controls(cfg4, 1, 0.05)
    for strang in (False, True):
        z[f"unitary4_{int(strang)}"] = trotter.PerQubitPlan(cfg4, 0.05, strang=strang).step_unitary(bx[0], by[0])

    replays = [
        ("r3", 3, (0.2,), 0.05, 40, 1, False),
        ("r4s", 4, (0.2,), 0.05, 200, 10, True),
        ("r5", 5, (0.2, 0.1), 0.1, 250, 25, False),
        ("r6", 6, (0.2,), 0.05, 500, 50, False),
        ("r8", 8, (0.2,), 0.05, 2000, 100, False),
    ] + [(f"c8n{n}", n, (0.2,), 0.05, 20000, 100, False) for n in range(3, 7)]
    names = []
    for name, n, cpl, tau, steps, rec, strang in replays:
        t0 = time.perf_counter()
        cfg = model.ModelConfig(n, 1.0, cpl, "per-qubit")
        z[f"{name}_fids"] = trotter.fidelity_replay(cfg, tau, steps, record_every=rec, strang=strang)
        z[f"{name}_spec"] = np.array([n, tau, steps, rec, int(strang)], dtype=np.float64)
        z[f"{name}_cpl"] = np.array(cpl)
        names.append(name)
        print(name, f"{time.perf_counter() - t0:.1f} s", flush=True)
    z["replays"] = np.array(names)
    slopes = []
    cfg3 = model.ModelConfig(3, 1.0, (0.2,), "per-qubit")
    for tau in (0.1, 0.05, 0.025):
        slopes.append(1.0 - trotter.fidelity_replay(cfg3, tau, int(round(25.0 / tau)), record_every=10**6)[-1])
    z["order_errs_n3"] = np.array(slopes)
    np.savez_compressed(OUT, **z)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
