"""Batched device-resident L-BFGS (optim.py) on CPU tensors."""

import numpy as np
import torch

from oracle import grape_oracle as O
from paper_2309_05884_b200 import optim, systems


def test_batched_lbfgs_solves_independent_quadratics():
    torch.manual_seed(0)
    B, n = 6, 12
    A = torch.randn(B, n, n, dtype=torch.float64)
    A = A @ A.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64)
    c = torch.randn(B, n, dtype=torch.float64)

    def fun(u, rows=None):  # maximise F = -(1/2 u^T A u - c^T u), a different quadratic per row
        rows = torch.arange(u.shape[0]) if rows is None else rows
        Au = torch.einsum("bij,bj->bi", A[rows], u)
        return -(0.5 * (u * Au).sum(1) - (c[rows] * u).sum(1)), -(Au - c[rows])

    res = optim.lbfgs_maximize(fun, torch.zeros(B, n, dtype=torch.float64), iterations=60, indexed=True)
    ustar = torch.linalg.solve(A, c)
    assert torch.allclose(res.u, ustar, atol=1e-6)
    assert all(b >= a - 1e-12 for a, b in zip(res.history, res.history[1:]))


def test_batched_lbfgs_on_grape_matches_per_seed_monotone_ascent():
    s = systems.config(0, n_slices=20)
    u0 = torch.from_numpy(s.controls(3, batch=3))

    def fun(u):
        F, g = [], []
        for b in range(u.shape[0]):
            f, gr, _ = O.objective(s, u[b].numpy())
            F.append(f)
            g.append(gr)
        return torch.tensor(F, dtype=torch.float64), torch.from_numpy(np.stack(g))

    res = optim.lbfgs_maximize(fun, u0, iterations=8)
    F0, _ = fun(u0)
    assert torch.all(res.F > F0)
    assert all(b >= a - 1e-12 for a, b in zip(res.history, res.history[1:]))
