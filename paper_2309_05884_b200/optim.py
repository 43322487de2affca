"""Device-resident batched L-BFGS for many independent GRAPE problems.

Maximises F_b(u_b) for every control vector b of a batch at once (cfg 1: 4096 seeds), with
all optimiser state -- iterates, gradients, the (s, y) history, the two-loop recursion and
the Armijo backtracking -- kept as torch tensors on the engine's device.  Each iteration is
one batched fidelity+gradient evaluation plus as many batched trial evaluations as the
slowest seed's line search needs; no per-seed host round trip.

The per-seed algorithm is textbook L-BFGS (two-loop recursion, history m, curvature check
s.y > 0) on -F with an Armijo backtracking line search (c = 1e-4, shrink 0.5, as the
reference's driver uses, qoc.py:25-27, 196-205).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch


@dataclass
class BatchedResult:
    u: torch.Tensor
    F: torch.Tensor
    history: list = field(default_factory=list)  # mean F per iteration
    evaluations: int = 0


class DeviceObjective:
    """F, grad for a (B, K, N) batch of device controls through GrapeEngine.evaluate_device."""

    def __init__(self, engine):
        self.engine = engine

    def __call__(self, u: torch.Tensor):
        B = u.shape[0]
        u = u.contiguous()
        F = torch.empty(B, dtype=torch.float64, device=u.device)
        g = torch.empty_like(u)
        self.engine.evaluate_device(u.data_ptr(), B, F.data_ptr(), g.data_ptr(),
                                    stream=torch.cuda.current_stream(u.device).cuda_stream)
        return F, g


def lbfgs_maximize(fun, u0: torch.Tensor, iterations: int = 50, history: int = 10, c1: float = 1e-4,
                   shrink: float = 0.5, max_backtracks: int = 12, indexed: bool = False) -> BatchedResult:
    """Maximise fun(u) -> (F (B,), grad (B, ...)) independently for every batch row.

    Line-search trials are evaluated on compacted sub-batches; when the objective differs per
    row (``indexed=True``) it is called as fun(u_sub, rows) with the original row indices.
    """
    B = u0.shape[0]
    shape = u0.shape
    u = u0.clone().reshape(B, -1)
    n = u.shape[1]
    dev, dt = u.device, u.dtype

    def f(x):
        F, g = fun(x.reshape(shape))
        return -F, -g.reshape(B, -1)  # minimise -F

    fval, g = f(u)
    evals = 1
    S = torch.zeros(history, B, n, dtype=dt, device=dev)
    Y = torch.zeros(history, B, n, dtype=dt, device=dev)
    rho = torch.zeros(history, B, dtype=dt, device=dev)
    valid = torch.zeros(history, B, dtype=torch.bool, device=dev)
    hist = [(-fval).mean()]  # device scalars: no host sync per iteration (converted at the end)
    res = BatchedResult(u=u, F=-fval)
    for it in range(iterations):
        # two-loop recursion (per seed; invalid history slots contribute nothing)
        q = g.clone()
        alpha = torch.zeros(history, B, dtype=dt, device=dev)
        order = [(it - 1 - i) % history for i in range(history)]  # newest first
        for j in order:
            a = torch.where(valid[j], rho[j] * (S[j] * q).sum(1), torch.zeros((), dtype=dt, device=dev))
            alpha[j] = a
            q = q - a[:, None] * Y[j]
        newest = order[0]
        yy = (Y[newest] * Y[newest]).sum(1)
        gamma = torch.where(valid[newest] & (yy > 0), (S[newest] * Y[newest]).sum(1) / yy.clamp_min(1e-300),
                            torch.full((B,), 1.0, dtype=dt, device=dev))
        r = gamma[:, None] * q
        for j in reversed(order):
            b = torch.where(valid[j], rho[j] * (Y[j] * r).sum(1), torch.zeros((), dtype=dt, device=dev))
            r = r + (alpha[j] - b)[:, None] * S[j]
        d = -r
        slope = (g * d).sum(1)
        bad = slope >= 0  # not a descent direction: fall back to steepest descent
        d = torch.where(bad[:, None], -g, d)
        slope = torch.where(bad, -(g * g).sum(1), slope)
        if it == 0:  # scale the first step to unit length
            step = 1.0 / g.norm(dim=1).clamp_min(1e-300)
        else:
            step = torch.ones(B, dtype=dt, device=dev)
        # batched Armijo backtracking: trial points are evaluated only for the seeds that have
        # not accepted yet (compacted sub-batch), so a few stubborn seeds cost little
        # seeds whose predicted decrease is below rounding are converged: they stay put
        accepted = slope.abs() <= 1e-13 * fval.abs().clamp_min(1.0)
        u_new, f_new, g_new = u.clone(), fval.clone(), g.clone()
        for _ in range(max_backtracks):
            idx = torch.nonzero(~accepted).squeeze(1)
            if idx.numel() == 0:
                break
            trial = u[idx] + step[idx, None] * d[idx]
            sub = trial.reshape((idx.numel(),) + tuple(shape[1:]))
            Ft, Gt = fun(sub, idx) if indexed else fun(sub)
            ft, gt = -Ft, -Gt.reshape(idx.numel(), -1)
            evals += 1
            ok = ft <= fval[idx] + c1 * step[idx] * slope[idx]
            acc_idx = idx[ok]
            u_new[acc_idx] = trial[ok]
            f_new[acc_idx] = ft[ok]
            g_new[acc_idx] = gt[ok]
            accepted[acc_idx] = True
            step[idx[~ok]] *= shrink
        s = u_new - u
        y = g_new - g
        sy = (s * y).sum(1)
        slot = it % history
        good = accepted & (sy > 1e-300)
        S[slot] = torch.where(good[:, None], s, S[slot])
        Y[slot] = torch.where(good[:, None], y, Y[slot])
        rho[slot] = torch.where(good, 1.0 / sy.clamp_min(1e-300), rho[slot])
        # a rejected pair invalidates the slot: the pair left there from `history` iterations ago
        # would otherwise be taken as the newest one (two-loop order, gamma scaling)
        valid[slot] = good
        u, fval, g = u_new, f_new, g_new
        hist.append((-fval).mean())
    res.history = torch.stack(hist).tolist()
    res.u = u.reshape(shape)
    res.F = -fval
    res.evaluations = evals
    return res
