"""The Trotter oracle (oracle/trotter_oracle.py) against outputs of the reference itself
(tests/golden/r02_trotter.npz, made by tests/golden/make_trotter_golden.py from symqoc.trotter)."""

import os

import numpy as np
import pytest

from oracle import trotter_oracle as O

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "r02_trotter.npz"))


def test_expm_2x2_matches_reference():
    for h, t, want in zip(Z["expm_h"], Z["expm_tau"], Z["expm_out"]):
        np.testing.assert_allclose(O.expm_2x2(h, t), want, atol=1e-15)


@pytest.mark.parametrize("tag,cpl", [("a", (0.2,)), ("b", (0.2, 0.1))])
@pytest.mark.parametrize("strang", [False, True])
def test_apply_step_matches_reference(tag, cpl, strang):
    out = O.apply_step(Z[f"step_{tag}_psi"], 5, 1.0, cpl, 0.05, Z[f"step_{tag}_bx"], Z[f"step_{tag}_by"], strang)
    np.testing.assert_allclose(out, Z[f"step_{tag}_out_{int(strang)}"], atol=1e-15)


@pytest.mark.parametrize("strang", [False, True])
def test_step_unitary_matches_reference(strang):
    bx, by = O.benchmark_controls(4, 1.0, 1, 0.05)
    u = O.apply_step(np.eye(16, dtype=complex), 4, 1.0, (0.2,), 0.05, bx[0], by[0], strang)
    np.testing.assert_allclose(u, Z[f"unitary4_{int(strang)}"], atol=1e-15)


@pytest.mark.parametrize("name", ["r3", "r4s", "r5", "r6"])
def test_fidelity_replay_matches_reference(name):
    n, tau, steps, rec, strang = Z[f"{name}_spec"]
    f = O.fidelity_replay(int(n), 1.0, tuple(Z[f"{name}_cpl"]), float(tau), int(steps), record_every=int(rec),
                          strang=bool(strang))
    np.testing.assert_allclose(f, Z[f"{name}_fids"], atol=1e-13)
