"""CPU restatement of the reference's Trotterised per-qubit propagator.

TEST INFRASTRUCTURE ONLY: the checker for paper_2309_05884_b200/trotter.py's GPU path.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import it.

Restates, with numpy on dense index arithmetic instead of the reference's swap-permutation
matrices:

* expm_2x2                  /root/reference/pkg/src/symqoc/trotter.py:48-65 (closed form)
* PerQubitPlan.apply_step   trotter.py:68-152: for i = n..1 the coupling phase exp(-i tau/n H_cpl)
                            on the rows, then exp(-i tau h_i) on qubit i; Strang: i = 1..n with
                            tau/2 factors and half phases, then the mirror sweep
* fidelity_replay           trotter.py:196-225: W <- U_trotter (W U_exact^dag), the exact step by
                            the sparse Taylor applicator (trotter.py:183-193, stopping rule
                            max|term| < 1e-13 max(1, max|out|)); F = |Tr W|^2 / dim^2
* benchmark_controls        trotter.py:159-170

Model (reference model.py:59-92, per-qubit control mode): H = sum_i bz/2 Z_i
+ sum_k c_k/4 sum_i Z_i Z_{i+k} + sum_i (bx_i X_i + by_i Y_i)/2, site 1 = most significant bit
(pauli.py:158-160).  Pinned to the reference itself by tests/golden/make_trotter_golden.py.
"""

from __future__ import annotations

import math

import numpy as np


def site_bit(n: int, i: int) -> int:
    """Bit position of 1-based site i (site 1 = MSB; pauli.py:158-160)."""
    return n - i


def coupling_diagonal(n: int, couplings) -> np.ndarray:
    """diag of sum_k c_k/4 sum_{i=1..n} Z_i Z_{i+k} (ring, literal sums; model.py:59-71)."""
    x = np.arange(1 << n)
    out = np.zeros(1 << n)
    for k, c in enumerate(couplings, start=1):
        if c == 0.0:
            continue
        for i in range(1, n + 1):
            j = (i - 1 + k) % n + 1
            zi = 1 - 2 * ((x >> site_bit(n, i)) & 1)
            zj = 1 - 2 * ((x >> site_bit(n, j)) & 1)
            out += 0.25 * c * zi * zj
    return out


def field_diagonal(n: int, bz: float) -> np.ndarray:
    x = np.arange(1 << n)
    out = np.zeros(1 << n)
    for i in range(1, n + 1):
        out += 0.5 * bz * (1 - 2 * ((x >> site_bit(n, i)) & 1))
    return out


def expm_2x2(h: np.ndarray, tau: float) -> np.ndarray:
    """exp(-i tau h) for a Hermitian 2 x 2 h: phase e^{-i tau c0} times cos - i sin (n . sigma)."""
    c0 = 0.5 * (h[0, 0] + h[1, 1]).real
    v = np.array([h[0, 1].real, -h[0, 1].imag, 0.5 * (h[0, 0] - h[1, 1]).real])
    r = math.sqrt(float(v @ v))
    ph = np.exp(-1j * tau * c0)
    if r < 1e-300:
        return ph * np.eye(2, dtype=np.complex128)
    nx, ny, nz = v / r
    c, s = math.cos(tau * r), math.sin(tau * r)
    return ph * np.array([[c - 1j * s * nz, -1j * s * (nx - 1j * ny)],
                          [-1j * s * (nx + 1j * ny), c + 1j * s * nz]])


def factor_2x2(bz: float, bx: float, by: float, tau: float) -> np.ndarray:
    h = np.array([[0.5 * bz, 0.5 * (bx - 1j * by)], [0.5 * (bx + 1j * by), -0.5 * bz]])
    return expm_2x2(h, tau)


def apply_single(arr: np.ndarray, n: int, i: int, u: np.ndarray) -> np.ndarray:
    """u on site i of the row index (the reference's swap-to-last + block broadcast)."""
    m = 1 << site_bit(n, i)
    x = np.arange(arr.shape[0])
    lo = x[(x & m) == 0]
    hi = lo | m
    out = arr.copy()
    out[lo] = u[0, 0] * arr[lo] + u[0, 1] * arr[hi]
    out[hi] = u[1, 0] * arr[lo] + u[1, 1] * arr[hi]
    return out


def _phase(arr, ph):
    return arr * ph if arr.ndim == 1 else arr * ph[:, None]


def apply_step(arr, n, bz, couplings, tau, bx, by, strang=False):
    """One Trotter step on a state (dim,) or on the rows of a (dim, m) accumulator."""
    diag = coupling_diagonal(n, couplings)
    coupled = any(c != 0.0 for c in couplings)
    arr = np.asarray(arr, dtype=np.complex128)
    if strang:
        half = 0.5 * tau
        ph = np.exp(-1j * (0.5 * tau / n) * diag)
        for i in range(1, n + 1):
            arr = apply_single(arr, n, i, factor_2x2(bz, bx[i - 1], by[i - 1], half))
            if coupled:
                arr = _phase(arr, ph)
        for i in range(n, 0, -1):
            if coupled:
                arr = _phase(arr, ph)
            arr = apply_single(arr, n, i, factor_2x2(bz, bx[i - 1], by[i - 1], half))
        return arr
    ph = np.exp(-1j * (tau / n) * diag)
    for i in range(n, 0, -1):
        if coupled:
            arr = _phase(arr, ph)
        arr = apply_single(arr, n, i, factor_2x2(bz, bx[i - 1], by[i - 1], tau))
    return arr


def hamiltonian_action(v: np.ndarray, n: int, diag: np.ndarray, bx, by) -> np.ndarray:
    """H v for H = diag + sum_i (bx_i X_i + by_i Y_i) / 2 (column action, pauli.py:163-187)."""
    x = np.arange(1 << n)
    out = diag[:, None] * v if v.ndim == 2 else diag * v
    for i in range(1, n + 1):
        m = 1 << site_bit(n, i)
        b = (x >> site_bit(n, i)) & 1
        # P e_c = phase(c) e_{c ^ m}:  (P v)[r] = phase(r ^ m) v[r ^ m]
        ph = 0.5 * bx[i - 1] + 0.5 * by[i - 1] * (1j - 2j * b)
        src = x ^ m
        w = ph[src]
        out = out + (w[:, None] * v[src] if v.ndim == 2 else w * v[src])
    return out


def taylor_expm_apply(n, diag, bx, by, tau, b, tol=1e-13):
    """exp(-i tau H) b by the truncated Taylor series with the reference's stopping rule."""
    out = np.array(b, dtype=np.complex128, copy=True)
    term = out.copy()
    for k in range(1, 80):
        term = hamiltonian_action(term, n, diag, bx, by) * (-1j * tau / k)
        out += term
        if np.max(np.abs(term)) < tol * max(1.0, np.max(np.abs(out))):
            return out
    raise RuntimeError("Taylor series for the step exponential did not converge")


def benchmark_controls(n, bz, n_steps, tau, amplitude=0.05):
    t = (np.arange(n_steps) + 0.5) * tau
    bx = np.empty((n_steps, n))
    by = np.empty((n_steps, n))
    for i in range(1, n + 1):
        phi = 2.0 * np.pi * i / n
        bx[:, i - 1] = amplitude * np.cos(bz * t + phi)
        by[:, i - 1] = amplitude * np.sin(bz * t + phi)
    return bx, by


def fidelity_replay(n, bz, couplings, tau, n_steps, controls=None, record_every=1, strang=False):
    """Per-step |Tr(K_exact^dag K_trotter)/2^n|^2, tracking W = K_trotter K_exact^dag."""
    bx, by = benchmark_controls(n, bz, n_steps, tau) if controls is None else controls
    dim = 1 << n
    diag = field_diagonal(n, bz) + coupling_diagonal(n, couplings)
    w_acc = np.eye(dim, dtype=np.complex128)
    fids = np.empty(-(-n_steps // record_every))
    out = 0
    for j in range(n_steps):
        w_acc = taylor_expm_apply(n, diag, bx[j], by[j], tau, w_acc.conj().T).conj().T
        w_acc = apply_step(w_acc, n, bz, couplings, tau, bx[j], by[j], strang)
        if (j + 1) % record_every == 0 or j == n_steps - 1:
            fids[out] = abs(np.trace(w_acc)) ** 2 / dim**2
            out += 1
    return fids[:out]
