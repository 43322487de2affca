"""GPU parity of the fused tiny-block kernel (d <= 16) against the reference and the oracle.

Tolerances (BASELINE.json north_star): F within 1e-10 absolute, gradients within
1e-8 relative, norm-wise ||g_gpu - g_ref||_inf / ||g_ref||_inf.
"""

import numpy as np
import pytest

from oracle import grape_oracle as O
from paper_2309_05884_b200 import qoc, systems
from paper_2309_05884_b200.engine import GrapeEngine

pytestmark = pytest.mark.gpu
F_TOL = 1e-10
G_TOL = 1e-8


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300)


class Duck:
    def __init__(self, h0, hx, hy):
        self.h0, self.hx, self.hy = h0, hx, hy
        self.dim = h0.shape[0]

    def hamiltonian(self, bx, by):
        return self.h0 + bx * self.hx + by * self.hy


@pytest.mark.parametrize("key", ["ising2", "ising3", "nn4_full", "nn4_first_block_d", "cfg0"])
def test_reference_gradient_signature_matches_reference_outputs(golden, key):
    g = lambda k: golden[f"{key}_{k}"]  # noqa: E731
    bx, by = (g("u")[0], g("u")[1]) if f"{key}_u" in golden else (g("bx"), g("by"))
    gx, gy, p = qoc.gradient(g("psi0"), g("psif"), bx, by, Duck(g("h0"), g("hx"), g("hy")), float(g("tau")))
    assert abs(p - float(g("P"))) <= F_TOL
    ref = np.concatenate([g("gx"), g("gy")])
    assert rel(np.concatenate([gx, gy]), ref) <= G_TOL


def test_empty_grid_gives_empty_gradient(golden):
    g = lambda k: golden[f"ising2_{k}"]  # noqa: E731
    gx, gy, p = qoc.gradient(g("psi0"), g("psif"), np.zeros(0), np.zeros(0), Duck(g("h0"), g("hx"), g("hy")), 0.05)
    assert gx.size == 0 and gy.size == 0 and p == pytest.approx(0.0)


def test_cfg0_against_oracle():
    s = systems.config(0)
    eng = GrapeEngine(s, max_batch=4)
    u = s.controls(3, batch=4)
    F, g = eng.objective(u)
    for b in range(4):
        Fo, go, _ = O.objective(s, u[b])
        assert abs(F[b] - Fo) <= F_TOL
        assert rel(g[b], go) <= G_TOL


def test_cfg1_sectors_full_length_against_oracle():
    s = systems.config(1)  # n=12 all-to-all, 7 S_n sectors, N=1000
    B = 64
    eng = GrapeEngine(s, max_batch=B)
    u = s.controls(11, batch=B)
    F, g, tau = eng.evaluate(u, want_tau=True)
    for b in (0, B - 1):
        Fo, go, per_block = O.objective(s, u[b])
        assert abs(F[b] - Fo) <= F_TOL
        assert rel(g[b], go) <= G_TOL
        w = s.block_weights()
        np.testing.assert_allclose(w * np.abs(tau[b]) ** 2, per_block, atol=F_TOL)


def test_gate_d6_blocks_pinned_by_reference(golden):
    """Gate fidelity per D_6 block: F vs reference expm/unitary_fidelity, grad vs reference FD."""
    u, dt, probes = golden["gate6_u"], float(golden["gate6_dt"]), golden["gate6_probes"]

    class Sys:
        objective = "gate"
        n_slices = u.shape[1]

    for b in range(8):
        blk = type("B", (), {})()
        blk.h0 = golden[f"dn6_b{b}_h0"]
        blk.hk = [golden[f"dn6_b{b}_hx"], golden[f"dn6_b{b}_hy"]]
        sysm = Sys()
        sysm.blocks = [blk]
        sysm.targets = [golden[f"gate6_b{b}_V"]]
        sysm.dt = dt
        d = blk.h0.shape[0]
        sysm.block_weights = lambda d=d: np.array([1.0 / d**2])
        eng = GrapeEngine(sysm, max_batch=1)
        F, g = eng.objective(u)
        assert abs(F - float(golden[f"gate6_b{b}_F"])) <= F_TOL
        rms = np.sqrt(np.mean(g**2))
        for (k, j), fd in zip(probes, golden[f"gate6_b{b}_fd"]):
            assert abs(fd - g[k, j]) / max(abs(fd), abs(g[k, j]), rms, 1e-9) < 1e-6
        eng.close()


def test_d6_full_basis_gate_system_against_oracle():
    s = systems.gate_ring(6, 10.0, 60)
    eng = GrapeEngine(s, max_batch=2)
    u = s.controls(5, batch=2)
    F, g = eng.objective(u)
    for b in range(2):
        Fo, go, _ = O.objective(s, u[b])
        assert abs(F[b] - Fo) <= F_TOL
        assert rel(g[b], go) <= G_TOL


def test_deterministic_bits():
    s = systems.config(1, n_slices=200)
    eng = GrapeEngine(s, max_batch=40)
    u = s.controls(2, batch=40)
    F1, g1 = eng.objective(u)
    F2, g2 = eng.objective(u)
    assert np.array_equal(F1, F2) and np.array_equal(g1, g2)


def test_nonfinite_raises_floating_point_error():
    s = systems.config(0)
    eng = GrapeEngine(s, max_batch=1)
    u = np.full((2, s.n_slices), 1e200)
    with pytest.raises(FloatingPointError):
        eng.objective(u)
    with pytest.raises(ValueError):
        eng.objective(np.full((2, s.n_slices), np.nan))
    with pytest.raises(ValueError):
        eng.objective(np.zeros((3, s.n_slices)))


def test_lbfgs_driver_improves_cfg0():
    s = systems.config(0)
    eng = GrapeEngine(s, max_batch=1)
    u0 = s.controls(0)
    f0, _ = eng.objective(u0)
    res = qoc.optimize_lbfgs(eng, u0, maxiter=50)
    assert res.trace[-1] > f0


@pytest.mark.parametrize("schedule", ["fused", "slice-parallel"])
@pytest.mark.parametrize("cfg,kw,batch", [(0, {}, 3), (1, {"n_slices": 120}, 5), (2, {"n": 6, "n_slices": 30}, 2)])
def test_tiny_schedules_against_oracle(schedule, cfg, kw, batch):
    s = systems.config(cfg, **kw)
    eng = GrapeEngine(s, max_batch=batch)
    eng.set_tiny_schedule(schedule)
    u = s.controls(8, batch=batch)
    F, g = eng.objective(u)
    assert eng.last_tiny_schedule == schedule
    for b in range(batch):
        Fo, go, _ = O.objective(s, u[b])
        assert abs(F[b] - Fo) <= F_TOL
        assert rel(g[b], go) <= G_TOL


def test_slice_parallel_is_the_default_for_single_evaluations():
    s = systems.config(0)
    eng = GrapeEngine(s, max_batch=1)
    eng.objective(s.controls(0))
    assert eng.last_tiny_schedule == "slice-parallel"


def test_integration_md_ctypes_stub_runs(golden):
    """The reference-side binding shown in INTEGRATION.md works as written."""
    import os
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    code = re.search(r"## 2\..*?```python\n(.*?)```", text, re.S).group(1)
    code = code.replace("/path/to/libsymqoc_b200.so", os.path.join(root, "paper_2309_05884_b200", "libsymqoc_b200.so"))
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    g = lambda k: golden[f"cfg0_{k}"]  # noqa: E731
    gx, gy, p = ns["gradient"](g("psi0"), g("psif"), g("u")[0], g("u")[1], Duck(g("h0"), g("hx"), g("hy")), 0.1)
    assert abs(p - float(g("P"))) <= F_TOL
    assert rel(np.concatenate([gx, gy]), np.concatenate([g("gx"), g("gy")])) <= G_TOL


def test_batched_device_lbfgs_improves_every_seed():
    import torch

    from paper_2309_05884_b200 import optim

    s = systems.config(1, n_slices=100)
    eng = GrapeEngine(s, max_batch=64)
    u0 = torch.from_numpy(s.controls(1, batch=64)).cuda()
    fun = optim.DeviceObjective(eng)
    F0, _ = fun(u0)
    res = optim.lbfgs_maximize(fun, u0, iterations=10)
    assert bool(torch.all(res.F >= F0))
    assert res.history[-1] > res.history[0] + 1e-3
    assert all(b >= a - 1e-12 for a, b in zip(res.history, res.history[1:]))


def test_tiny_cta_size_does_not_change_results():
    """sqoc_set_tiny_cta_warps only regroups problems into CTAs: bit-identical F and gradient."""
    import copy

    import numpy as np

    from paper_2309_05884_b200 import systems
    from paper_2309_05884_b200.engine import GrapeEngine

    multi = systems.config(1, n=8, n_slices=40)
    single = copy.copy(multi)
    single.blocks, single.targets = [multi.blocks[0]], [multi.targets[0]]
    for s in (multi, single):
        u = s.controls(11, batch=75)
        eng = GrapeEngine(s, max_batch=75)
        eng.set_tiny_schedule("fused")
        ref = None
        for w in (-1, 0, 3, 1):
            eng.set_tiny_cta_warps(w)
            F, g = eng.objective(u)
            if ref is None:
                ref = (F.copy(), g.copy())
            else:
                assert np.array_equal(F, ref[0]) and np.array_equal(g, ref[1])
        eng.close()
