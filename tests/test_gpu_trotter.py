"""GPU Trotterised per-qubit propagator (csrc/trotter.cu through the C ABI) against the reference's
own outputs (tests/golden/r02_trotter.npz: symqoc.trotter, trotter.py:48-225) and the reference's
acceptance properties (test_trotter.py, test_acceptance.py:212-250).

Tolerances: states / unitaries 1e-13 absolute; fidelities 1e-10 absolute (north_star's fidelity bar).
"""

import os

import numpy as np
import pytest

from oracle import trotter_oracle as O
from paper_2309_05884_b200 import trotter

pytestmark = pytest.mark.gpu

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "r02_trotter.npz"))
TROTTER_MIN_FIDELITY = 0.996  # test_acceptance.py:25


@pytest.mark.parametrize("tag,cpl", [("a", (0.2,)), ("b", (0.2, 0.1))])
@pytest.mark.parametrize("strang", [False, True])
def test_apply_step_matches_reference(tag, cpl, strang):
    plan = trotter.PerQubitPlan(trotter.TrotterModel(5, 1.0, cpl), 0.05, strang=strang)
    out = plan.apply_step(Z[f"step_{tag}_psi"], Z[f"step_{tag}_bx"], Z[f"step_{tag}_by"])
    np.testing.assert_allclose(out, Z[f"step_{tag}_out_{int(strang)}"], atol=1e-13)
    plan.close()


@pytest.mark.parametrize("strang", [False, True])
def test_step_unitary_matches_reference(strang):
    cfg = trotter.TrotterModel(4, 1.0, (0.2,))
    bx, by = trotter.benchmark_controls(cfg, 1, 0.05)
    plan = trotter.PerQubitPlan(cfg, 0.05, strang=strang)
    np.testing.assert_allclose(plan.step_unitary(bx[0], by[0]), Z[f"unitary4_{int(strang)}"], atol=1e-13)


@pytest.mark.parametrize("name", [str(x) for x in Z["replays"]])
def test_fidelity_replay_matches_reference(name):
    n, tau, steps, rec, strang = Z[f"{name}_spec"]
    cfg = trotter.TrotterModel(int(n), 1.0, tuple(Z[f"{name}_cpl"]))
    f = trotter.fidelity_replay(cfg, float(tau), int(steps), record_every=int(rec), strang=bool(strang))
    np.testing.assert_allclose(f, Z[f"{name}_fids"], atol=1e-10, rtol=0)


def test_many_steps_on_chip_equal_repeated_single_steps_and_oracle():
    """apply_steps runs every step inside one launch; it equals step-by-step application and the oracle."""
    cfg = trotter.TrotterModel(7, 1.0, (0.2, 0.05))
    rng = np.random.default_rng(3)
    bx = rng.uniform(-1, 1, (30, 7))
    by = rng.uniform(-1, 1, (30, 7))
    a0 = rng.standard_normal((128, 5)) + 1j * rng.standard_normal((128, 5))
    for strang in (False, True):
        plan = trotter.PerQubitPlan(cfg, 0.07, strang=strang)
        fused = plan.apply_steps(a0, bx, by)
        step = a0
        ref = a0
        for j in range(30):
            step = plan.apply_step(step, bx[j], by[j])
            ref = O.apply_step(ref, 7, 1.0, (0.2, 0.05), 0.07, bx[j], by[j], strang)
        np.testing.assert_allclose(fused, step, atol=1e-13)
        np.testing.assert_allclose(fused, ref, atol=1e-12)


@pytest.mark.parametrize("n", [3, 8, 12])
def test_step_unitarity(n):
    cfg = trotter.TrotterModel(n, 1.0, (0.2,))
    bx, by = trotter.benchmark_controls(cfg, 1, 0.05)
    k = trotter.PerQubitPlan(cfg, 0.05).step_unitary(bx[0], by[0])
    np.testing.assert_allclose(k.conj().T @ k, np.eye(1 << n), atol=1e-12)


def test_uncoupled_plan_is_exact():
    """Without coupling the factors commute: one step equals exp(-i tau H) (test_trotter.py:71-80)."""
    cfg = trotter.TrotterModel(3, 1.0, ())
    bx, by = trotter.benchmark_controls(cfg, 1, 0.3)
    got = trotter.PerQubitPlan(cfg, 0.3).step_unitary(bx[0], by[0])
    diag = O.field_diagonal(3, 1.0)
    want = O.taylor_expm_apply(3, diag, bx[0], by[0], 0.3, np.eye(8, dtype=complex), tol=1e-17)
    np.testing.assert_allclose(got, want, atol=1e-12)


def test_error_order_matches_reference_and_slope():
    cfg = trotter.TrotterModel(3, 1.0, (0.2,))
    errs = [1.0 - trotter.fidelity_replay(cfg, tau, int(round(25.0 / tau)), record_every=10**6)[-1]
            for tau in (0.1, 0.05, 0.025)]
    np.testing.assert_allclose(errs, Z["order_errs_n3"], atol=1e-10)
    slope = np.polyfit(np.log([0.1, 0.05, 0.025]), np.log(errs), 1)[0]
    assert 1.8 <= slope <= 2.3


def test_acceptance_criterion_8_fidelity_floor_n3_to_11():
    """test_acceptance.py:212-235 (n = 3..8, and the opt-in n = 11): min F over 20000 steps >= 0.996."""
    for n in (3, 5, 8, 11):
        cfg = trotter.TrotterModel(n, 1.0, (0.2,))
        f = trotter.fidelity_replay(cfg, 0.05, 20000, record_every=100)
        assert f.shape == (200,)
        assert f.min() >= TROTTER_MIN_FIDELITY, (n, f.min())


def test_plan_errors():
    with pytest.raises(ValueError):
        trotter.PerQubitPlan(trotter.TrotterModel(3, 1.0, (0.2,), "global"), 0.05)
    with pytest.raises(ValueError):
        trotter.PerQubitPlan(trotter.TrotterModel(13, 1.0, ()), 0.05)
    with pytest.raises(ValueError):
        trotter.PerQubitPlan(trotter.TrotterModel(4, 1.0, (0.2, 0.1, 0.1)), 0.05)
    plan = trotter.PerQubitPlan(trotter.TrotterModel(3, 1.0, (0.2,)), 0.05)
    with pytest.raises(ValueError):
        plan.apply_step(np.ones(8, dtype=complex), np.zeros(2), np.zeros(3))
