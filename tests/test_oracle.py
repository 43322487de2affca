"""The CPU oracle against outputs of the reference package itself (tests/golden)."""

import numpy as np
import pytest

from oracle import grape_oracle as O


def _state_case(g, key):
    f = lambda k: g[f"{key}_{k}"]  # noqa: E731
    if f"{key}_u" in g:
        bx, by = f("u")[0], f("u")[1]
    else:
        bx, by = f("bx"), f("by")
    return f("h0"), f("hx"), f("hy"), f("psi0"), f("psif"), bx, by, float(f("tau")), f("gx"), f("gy"), float(f("P"))


@pytest.mark.parametrize("key", ["ising2", "ising3", "nn4_full", "nn4_first_block_d", "cfg0"])
def test_state_gradient_matches_reference(golden, key):
    h0, hx, hy, psi0, psif, bx, by, tau, gx, gy, P = _state_case(golden, key)
    grad, _, p = O.state_gradient(psi0, psif, np.stack([bx, by]), h0, [hx, hy], tau)
    # same algorithm, same LAPACK: agreement at rounding level
    assert abs(p - P) <= 1e-13
    scale = max(np.abs(gx).max(), np.abs(gy).max())
    assert np.abs(grad[0] - gx).max() <= 1e-12 * scale
    assert np.abs(grad[1] - gy).max() <= 1e-12 * scale


def test_block_gradient_equals_full_gradient(golden):
    """test_qoc.py:84-99: first-block-d gradients equal the full-space ones."""
    a = golden["nn4_full_gx"], golden["nn4_full_gy"], golden["nn4_full_P"]
    b = golden["nn4_first_block_d_gx"], golden["nn4_first_block_d_gy"], golden["nn4_first_block_d_P"]
    np.testing.assert_allclose(a[0], b[0], atol=1e-8)
    np.testing.assert_allclose(a[1], b[1], atol=1e-8)
    assert abs(float(a[2]) - float(b[2])) <= 1e-10


def test_gate_fidelity_and_gradient_pinned_by_reference(golden):
    """F_b via reference expm_hermitian + unitary_fidelity; dF_b/du via central FD of it."""
    u, dt, probes = golden["gate6_u"], float(golden["gate6_dt"]), golden["gate6_probes"]
    b = 0
    while f"dn6_b{b}_h0" in golden:
        h0, hx, hy = golden[f"dn6_b{b}_h0"], golden[f"dn6_b{b}_hx"], golden[f"dn6_b{b}_hy"]
        V = golden[f"gate6_b{b}_V"]
        d = h0.shape[0]
        tr, dtau = O.gate_dtau(V, u, h0, [hx, hy], dt)
        F = abs(tr) ** 2 / d**2
        assert abs(F - float(golden[f"gate6_b{b}_F"])) <= 1e-12
        grad = 2.0 * np.real(np.conj(tr) * dtau) / d**2
        fd = golden[f"gate6_b{b}_fd"]
        rms = np.sqrt(np.mean(grad**2))
        for (k, j), f in zip(probes, fd):
            assert abs(f - grad[k, j]) / max(abs(f), abs(grad[k, j]), rms, 1e-9) < 1e-6
        b += 1
    assert b == 8


def test_frechet_weights_degenerate_branch():
    w = np.array([0.3, 0.3, 1.2])
    g = O.frechet_weights(w, 0.1)
    f = np.exp(-1j * 0.1 * w)
    assert g[0, 1] == pytest.approx(-1j * 0.1 * f[0])
    assert g[0, 2] == pytest.approx((f[0] - f[2]) / (w[0] - w[2]))


def test_state_dtau_consistent_with_state_gradient(golden):
    h0, hx, hy, psi0, psif, bx, by, tau, gx, gy, P = _state_case(golden, "cfg0")
    o, dtau = O.state_dtau(psi0, psif, np.stack([bx, by]), h0, [hx, hy], tau)
    grad = 2 * np.real(np.conj(o) * dtau)
    np.testing.assert_allclose(grad[0], gx, atol=1e-12)
    np.testing.assert_allclose(grad[1], gy, atol=1e-12)


def test_r02_cfg1_fixture_reproduces_with_current_systems():
    """The cfg 1 fixture (tests/golden/make_fixtures_r02.py) is reproducible from the current host
    systems: same inputs (checksum) and the same oracle output on its first row."""
    import os

    from paper_2309_05884_b200 import systems

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "r02_cfg1.npz"))
    s = systems.config(1)
    ub = s.controls(0, batch=4096)
    rows = list(z["cfg1_rows"])
    chk = []
    for a in (ub[rows], *s.targets, *[b.h0 for b in s.blocks]):
        a = np.asarray(a).astype(np.complex128).ravel()
        w = np.arange(1, a.size + 1, dtype=np.float64)
        chk += [a.sum(), (w * a).sum() / a.size]
    np.testing.assert_allclose(np.array(chk), z["cfg1_check"], rtol=1e-10, atol=1e-12)
    F, g, _ = O.objective(s, ub[rows[0]])
    assert abs(F - z["cfg1_F"][0]) <= 1e-12
    assert np.abs(g - z["cfg1_grad"][0]).max() <= 1e-10 * np.abs(g).max()
