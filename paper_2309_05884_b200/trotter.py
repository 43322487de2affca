"""Trotterised per-qubit propagator on the GPU.

Host mirror of the reference's ``symqoc.trotter`` per-qubit path
(/root/reference/pkg/src/symqoc/trotter.py): ``PerQubitPlan`` (:68-152), ``fidelity_replay``
(:196-225), ``benchmark_controls`` (:159-170) and ``expm_2x2`` (:48-65), with the same names,
argument meanings and errors.  The step, the exact-step Taylor applicator and the fidelity trace
run in ``csrc/trotter.cu`` through the C ABI (``sqoc_trotter_*``); there is no CPU path.

``cfg`` is any object with ``n``, ``bz``, ``couplings`` and ``control_mode`` -- the reference's
``model.ModelConfig`` or ``TrotterModel`` below.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class TrotterModel:
    """The reference's ModelConfig fields the Trotter path reads (model.py:22-44)."""

    n: int
    bz: float = 1.0
    couplings: tuple = ()
    control_mode: str = "per-qubit"

    @property
    def coupled(self) -> bool:
        return any(c != 0.0 for c in self.couplings)


def expm_2x2(h: np.ndarray, tau: float) -> np.ndarray:
    """exp(-i tau H) for a 2 x 2 Hermitian H in closed form (trotter.py:48-65; host helper)."""
    c0 = 0.5 * (h[0, 0] + h[1, 1]).real
    vx, vy, vz = h[0, 1].real, -h[0, 1].imag, 0.5 * (h[0, 0] - h[1, 1]).real
    r = math.sqrt(vx * vx + vy * vy + vz * vz)
    phase = np.exp(-1j * tau * c0)
    if r < 1e-300:
        return phase * np.eye(2, dtype=np.complex128)
    c, s = math.cos(tau * r), math.sin(tau * r)
    nx, ny, nz = vx / r, vy / r, vz / r
    return phase * np.array([[c - 1j * s * nz, -1j * s * (nx - 1j * ny)],
                             [-1j * s * (nx + 1j * ny), c + 1j * s * nz]])


def benchmark_controls(cfg, n_steps: int, tau: float, amplitude: float = 0.05):
    """Pinned per-qubit drive: phase-staggered resonant tones (trotter.py:159-170)."""
    t = (np.arange(n_steps) + 0.5) * tau
    n = cfg.n
    bx = np.empty((n_steps, n))
    by = np.empty((n_steps, n))
    for i in range(1, n + 1):
        phi = 2.0 * np.pi * i / n
        bx[:, i - 1] = amplitude * np.cos(cfg.bz * t + phi)
        by[:, i - 1] = amplitude * np.sin(cfg.bz * t + phi)
    return bx, by


def _controls(n: int, bx, by, steps: int | None = None):
    bx = np.ascontiguousarray(np.asarray(bx, dtype=np.float64))
    by = np.ascontiguousarray(np.asarray(by, dtype=np.float64))
    if bx.shape != by.shape or bx.shape[-1] != n or (steps is not None and bx.reshape(-1, n).shape[0] != steps):
        raise ValueError("need one control pair per qubit")
    return bx, by


class PerQubitPlan:
    """The transformed Trotter plan for a ring with per-qubit controls (trotter.py:68-152) on a GPU.

    One step applies, for i = n..1, exp(-i (tau/n) H_cpl) and then exp(-i tau h_i) on site i;
    with ``strang`` the second-order splitting (tau/2 sweep i = 1..n, then the mirror sweep).
    """

    def __init__(self, cfg, tau: float, strang: bool = False, device: int = 0):
        if cfg.control_mode != "per-qubit":
            raise ValueError("per-qubit plan needs control_mode='per-qubit'")
        self.cfg = cfg
        self.n = cfg.n
        self.tau = tau
        self.strang = strang
        self.dim = 1 << cfg.n
        self.lib = _lib.load()
        cpl = np.ascontiguousarray(np.asarray(cfg.couplings, dtype=np.float64))
        h = ctypes.c_void_p()
        _lib.check(self.lib.sqoc_trotter_create(ctypes.byref(h), device, cfg.n, float(cfg.bz),
                                                cpl.ctypes.data if cpl.size else None, int(cpl.size), float(tau),
                                                1 if strang else 0), "sqoc_trotter_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sqoc_trotter_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def factor_2x2(self, bx: float, by: float, tau: float | None = None) -> np.ndarray:
        h = np.array([[0.5 * self.cfg.bz, 0.5 * (bx - 1j * by)], [0.5 * (bx + 1j * by), -0.5 * self.cfg.bz]])
        return expm_2x2(h, self.tau if tau is None else tau)

    @property
    def last_launches(self) -> int:
        return self.lib.sqoc_trotter_last_launches(self.handle)

    def apply_steps(self, arr: np.ndarray, bx, by) -> np.ndarray:
        """len(bx) Trotter steps (controls (steps, n)) on a state (dim,) or the rows of (dim, m)."""
        a = np.array(arr, dtype=np.complex128, order="C", copy=True)
        if a.shape[0] != self.dim or a.ndim not in (1, 2):
            raise ValueError(f"need a state or accumulator with {self.dim} rows, got {a.shape}")
        bx, by = _controls(self.n, bx, by)
        steps = bx.reshape(-1, self.n).shape[0]
        cols = 1 if a.ndim == 1 else a.shape[1]
        _lib.check(self.lib.sqoc_trotter_apply(self.handle, a.ctypes.data, cols, bx.ctypes.data, by.ctypes.data,
                                               steps, _lib.MEM_HOST, None), "sqoc_trotter_apply")
        return a

    def apply_step(self, arr: np.ndarray, bx, by) -> np.ndarray:
        """One Trotter step applied to a state vector or unitary accumulator (trotter.py:138-152)."""
        if len(bx) != self.n or len(by) != self.n:
            raise ValueError("need one control pair per qubit")
        return self.apply_steps(arr, np.asarray(bx)[None], np.asarray(by)[None])

    def step_unitary(self, bx, by) -> np.ndarray:
        return self.apply_step(np.eye(self.dim, dtype=np.complex128), bx, by)

    def replay(self, bx, by, record_every: int = 1) -> np.ndarray:
        """Per-step |Tr(K_exact^dag K_trotter)/2^n|^2 for controls (steps, n) (trotter.py:196-225)."""
        bx, by = _controls(self.n, bx, by)
        steps = bx.shape[0]
        n_rec = -(-steps // record_every)
        fids = np.empty(n_rec)
        _lib.check(self.lib.sqoc_trotter_replay(self.handle, bx.ctypes.data, by.ctypes.data, steps,
                                                int(record_every), fids.ctypes.data, _lib.MEM_HOST, None),
                   "sqoc_trotter_replay")
        return fids

    def replay_device(self, bx_ptr: int, by_ptr: int, steps: int, record_every: int, fids_ptr: int,
                      stream: int = 0) -> None:
        """Device pointers (e.g. torch data_ptr()); blocking."""
        _lib.check(self.lib.sqoc_trotter_replay(self.handle, bx_ptr, by_ptr, int(steps), int(record_every), fids_ptr,
                                                _lib.MEM_DEVICE, stream or None), "sqoc_trotter_replay")


def plan_per_qubit_coupled(cfg, tau: float) -> PerQubitPlan:
    return PerQubitPlan(cfg, tau)


def fidelity_replay(cfg, tau: float, n_steps: int, controls=None, record_every: int = 1,
                    strang: bool = False, device: int = 0) -> np.ndarray:
    """Per-step unitary fidelities |Tr(K_exact^+ K_trotter)/2^n|^2 (trotter.py:196-225).

    Tracks W = K_trotter K_exact^+ on the GPU: each step right-multiplies by the inverse exact
    step (Taylor series of the sparse H, row by row) and left-multiplies by the Trotter step.
    """
    plan = PerQubitPlan(cfg, tau, strang=strang, device=device)
    try:
        bx, by = benchmark_controls(cfg, n_steps, tau) if controls is None else controls
        return plan.replay(np.asarray(bx)[:n_steps], np.asarray(by)[:n_steps], record_every)
    finally:
        plan.close()
