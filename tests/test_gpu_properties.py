"""Size-independent properties at the BASELINE sizes (where the oracle is too slow to run)."""

import numpy as np
import pytest

from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    s = systems.config(1)  # n=12 all-to-all, 7 sectors, N=1000
    eng = GrapeEngine(s, max_batch=4096)  # auto histories: up to ~70% of free device memory
    u = s.controls(31, batch=4096)
    F, g, tau = eng.evaluate(u, want_tau=True)
    yield s, eng, u, F, g, tau
    eng.close()  # release the histories before the full-size large-block tests


def test_cfg1_fidelity_bounds_and_tau(cfg1):
    s, eng, u, F, g, tau = cfg1
    assert np.all(np.isfinite(F)) and np.all(F >= 0) and np.all(F <= 1 + 1e-12)
    assert np.all(np.isfinite(g))
    # |tau_b| <= d_b for unitary propagators and unitary targets (Cauchy-Schwarz)
    dims = np.array([b.dim for b in s.blocks])
    assert np.all(np.abs(tau) <= dims[None, :] * (1 + 1e-12))
    np.testing.assert_allclose(F, (s.block_weights()[None, :] * np.abs(tau) ** 2).sum(1), rtol=1e-14, atol=1e-15)


def test_cfg1_batch_permutation_equivariance(cfg1):
    s, eng, u, F, g, tau = cfg1
    perm = np.random.default_rng(0).permutation(4096)
    F2, g2 = eng.objective(u[perm])
    # results of a seed do not depend on its batch position or neighbours beyond rounding
    np.testing.assert_allclose(F2, F[perm], rtol=0, atol=1e-13)
    np.testing.assert_allclose(g2, g[perm], rtol=0, atol=1e-11 * np.abs(g).max())


def test_cfg1_directional_derivative(cfg1):
    s, eng, u, F, g, tau = cfg1
    rng = np.random.default_rng(1)
    idx = [0, 1234, 4095]
    du = rng.standard_normal((len(idx),) + u.shape[1:])
    h = 1e-5
    Fp, _ = eng.objective(u[idx] + h * du)
    Fm, _ = eng.objective(u[idx] - h * du)
    fd = (Fp - Fm) / (2 * h)
    an = np.einsum("bkn,bkn->b", g[idx], du)
    np.testing.assert_allclose(fd, an, rtol=1e-6, atol=1e-9)


def test_cfg1_target_phase_invariance():
    s = systems.config(1, n_slices=200)
    u = s.controls(3, batch=16)
    F, g = GrapeEngine(s, max_batch=16).objective(u)
    s.targets = [np.exp(1j * 0.7 * (b + 1)) * t for b, t in enumerate(s.targets)]
    F2, g2 = GrapeEngine(s, max_batch=16).objective(u)
    np.testing.assert_allclose(F2, F, atol=1e-14)
    np.testing.assert_allclose(g2, g, atol=1e-12 * np.abs(g).max())


def test_cfg1_release(cfg1):
    """Free the module's cfg 1 engine (tens of GB of histories) before the full-size cfg 2/4 tests."""
    cfg1[1].close()


def test_cfg2_full_size_schedules_agree_and_gauge():
    s = systems.config(2)
    eng = GrapeEngine(s, max_batch=1)
    u = s.controls(4)
    F1, g1 = eng.objective(u)
    eng.set_schedule("sequential")
    F2, g2 = eng.objective(u)
    assert abs(F1 - F2) <= 1e-12
    assert np.abs(g1 - g2).max() <= 1e-9 * np.abs(g1).max()
    assert 0 <= F1 <= 1


@pytest.mark.slow
def test_cfg4_full_size_matrix_free_equals_dense_state_vector():
    """cfg 4 at full size: the dense DMMA state-vector schedule and the matrix-free schedule agree."""
    s = systems.config(4)
    eng = GrapeEngine(s, max_batch=1)
    u = s.controls(0)
    eng.set_schedule("matrix-free")
    F1, g1 = eng.objective(u)
    eng.set_schedule("state-vector")
    F2, g2 = eng.objective(u)
    assert abs(F1 - F2) <= 1e-10
    assert np.abs(g1 - g2).max() <= 1e-8 * np.abs(g2).max()


def test_cfg4_symmetric_equals_conventional_at_full_size():
    """The paper's central claim at the BASELINE size: n=12, N=200 state transfer in the full
    4096-dim space (matrix-free schedule) equals the same evaluation in the 224-dim A1 block."""
    full = systems.config(4)
    blk = systems.config(4, full=False)
    u = full.controls(2)
    ef = GrapeEngine(full, max_batch=1)
    ef.set_schedule("matrix-free")
    Ff, gf = ef.objective(u)
    Fb, gb = GrapeEngine(blk, max_batch=1).objective(u)
    assert abs(Ff - Fb) <= 1e-10
    assert np.abs(gf - gb).max() <= 1e-8 * np.abs(gb).max()
