"""NumPy restatement of the reference's fidelity+gradient evaluation (test infrastructure).

State transfer restates ``symqoc.qoc.gradient`` (``pkg/src/symqoc/qoc.py:137-168``)
line by line: eigendecomposition propagators (``propagate.py:48-53``), forward
states (``qoc.py:128-134``), backward costates, and exact Daleckii-Krein
derivatives (``qoc.py:115-125``), generalised from (bx, by) to K controls.

The gate-fidelity objective has no gradient in the reference (SURVEY.md
section 8c gap G2).  It is restated on the same primitives: per block
tau_b = Tr(V_b^dagger X_N) with X_N = U_N ... U_1, F_b = |tau_b|^2 / d_b^2
(``propagate.unitary_fidelity``, ``propagate.py:161-167``), and

    d tau_b / d u_kj = sum_pq (Q^dag X_{j-1} Lam_j^dag Q)_qp (G_j o Q^dag H_k Q)_pq,

with H_j = Q diag(w) Q^dag (eigh), G_j = frechet_weights(w, dt) and
Lam_j = U_{j+1}^dag ... U_N^dag V_b the backward-propagated target.

Objective over blocks: F = sum_b w_b |tau_b|^2 (w_b = 1/(N_B d_b^2) for gate
fidelity, 1 for state transfer) and dF/du = sum_b 2 w_b Re(conj(tau_b) dtau_b/du).
"""

from __future__ import annotations

import numpy as np

DEGENERACY_TOL = 1e-12  # qoc.py:120-123


def frechet_weights(w: np.ndarray, tau: float) -> np.ndarray:
    """Divided differences of f(x) = exp(-i tau x) (qoc.py:115-125)."""
    f = np.exp(-1j * tau * w)
    dw = w[:, None] - w[None, :]
    df = f[:, None] - f[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        g = np.where(np.abs(dw) > DEGENERACY_TOL, df / np.where(dw == 0, 1.0, dw), 0.0)
    same = np.abs(dw) <= DEGENERACY_TOL
    deriv = -1j * tau * f
    g[same] = 0.5 * (deriv[:, None] + deriv[None, :])[same]
    return g


def hamiltonian(h0, hk, u_j):
    """H = H0 + sum_k u_k H_k (propagate.py:88-89)."""
    h = h0.copy()
    for c, hc in zip(u_j, hk):
        h = h + c * hc
    return h


def expm_hermitian(h, tau):
    """exp(-i tau H) via eigh, plus the eigenpairs (propagate.py:48-53)."""
    w, v = np.linalg.eigh(h)
    return (v * np.exp(-1j * tau * w)) @ v.conj().T, (w, v)


def state_gradient(psi0, psi_f, u, h0, hk, tau):
    """(grad (K, N), overlap o, P = |o|^2) for one block (qoc.py:137-168)."""
    u = np.asarray(u, dtype=np.float64)
    n_steps = u.shape[1]
    states = np.empty((n_steps + 1, h0.shape[0]), dtype=np.complex128)
    states[0] = psi0
    for j in range(n_steps):  # qoc.py:128-134
        uj, _ = expm_hermitian(hamiltonian(h0, hk, u[:, j]), tau)
        states[j + 1] = uj @ states[j]
    overlap = np.vdot(psi_f, states[-1])
    grad = np.zeros(u.shape)
    chi = np.array(psi_f, dtype=np.complex128)
    for j in range(n_steps - 1, -1, -1):  # qoc.py:156-167
        w, v = np.linalg.eigh(hamiltonian(h0, hk, u[:, j]))
        g = frechet_weights(w, tau)
        vh = v.conj().T
        psi_eig = vh @ states[j]
        chi_eig = vh @ chi
        for k, hc in enumerate(hk):
            dpsi = (g * (vh @ hc @ v)) @ psi_eig
            grad[k, j] = 2.0 * np.real(np.conj(overlap) * np.vdot(chi_eig, dpsi))
        uj = (v * np.exp(-1j * tau * w)) @ vh
        chi = uj.conj().T @ chi
    return grad, overlap, float(abs(overlap) ** 2)


def state_dtau(psi0, psi_f, u, h0, hk, tau):
    """(tau = <psi_f|psi_N>, d tau / d u (K, N) complex) -- the complex form of state_gradient."""
    u = np.asarray(u, dtype=np.float64)
    n_steps = u.shape[1]
    states = np.empty((n_steps + 1, h0.shape[0]), dtype=np.complex128)
    states[0] = psi0
    for j in range(n_steps):
        uj, _ = expm_hermitian(hamiltonian(h0, hk, u[:, j]), tau)
        states[j + 1] = uj @ states[j]
    overlap = np.vdot(psi_f, states[-1])
    dtau = np.zeros(u.shape, dtype=np.complex128)
    chi = np.array(psi_f, dtype=np.complex128)
    for j in range(n_steps - 1, -1, -1):
        w, v = np.linalg.eigh(hamiltonian(h0, hk, u[:, j]))
        g = frechet_weights(w, tau)
        vh = v.conj().T
        psi_eig = vh @ states[j]
        chi_eig = vh @ chi
        for k, hc in enumerate(hk):
            dtau[k, j] = np.vdot(chi_eig, (g * (vh @ hc @ v)) @ psi_eig)
        chi = ((v * np.exp(-1j * tau * w)) @ vh).conj().T @ chi
    return overlap, dtau


def gate_dtau(target, u, h0, hk, tau, x0=None, lam_end=None):
    """(tau = Tr(V^dag X_N), d tau / d u (K, N) complex) for one block (gap G2).

    ``x0`` / ``lam_end`` override X_0 = I and Lam_N = V (slice-chunk boundaries).
    """
    u = np.asarray(u, dtype=np.float64)
    n_steps = u.shape[1]
    d = h0.shape[0]
    xs = np.empty((n_steps + 1, d, d), dtype=np.complex128)
    xs[0] = np.eye(d) if x0 is None else x0
    eig = []
    for j in range(n_steps):
        uj, (w, v) = expm_hermitian(hamiltonian(h0, hk, u[:, j]), tau)
        eig.append((w, v, uj))
        xs[j + 1] = uj @ xs[j]
    tr = np.vdot(target, xs[-1])  # Tr(V^dag X_N) = sum conj(V) * X_N
    dtau = np.zeros(u.shape, dtype=np.complex128)
    lam = np.array(target if lam_end is None else lam_end, dtype=np.complex128)
    for j in range(n_steps - 1, -1, -1):
        w, v, uj = eig[j]
        g = frechet_weights(w, tau)
        vh = v.conj().T
        bq = (vh @ xs[j]) @ (vh @ lam).conj().T  # Q^dag X_{j-1} Lam_j^dag Q
        for k, hc in enumerate(hk):
            dtau[k, j] = np.sum(bq.T * g * (vh @ hc @ v))
        lam = uj.conj().T @ lam
    return tr, dtau


def block_dtau(system, b, u):
    """(tau_b, dtau_b/du) for block b of a ``GrapeSystem`` with controls u (K, N)."""
    blk = system.blocks[b]
    if system.objective == "gate":
        return gate_dtau(system.targets[b], u, blk.h0, blk.hk, system.dt)
    return state_dtau(system.initial[b], system.targets[b], u, blk.h0, blk.hk, system.dt)


def objective(system, u, blocks=None):
    """F = sum_b w_b |tau_b|^2 and dF/du (K, N); also per-block |tau_b|^2 w_b.

    ``blocks`` restricts the sum to a subset (for sampled CPU timing).
    """
    w = system.block_weights()
    idx = range(len(system.blocks)) if blocks is None else blocks
    f_total = 0.0
    grad = np.zeros(np.shape(u))
    per_block = np.zeros(len(system.blocks))
    for b in idx:
        tr, dtau = block_dtau(system, b, u)
        per_block[b] = w[b] * abs(tr) ** 2
        f_total += per_block[b]
        grad += 2.0 * w[b] * np.real(np.conj(tr) * dtau)
    return f_total, grad, per_block


class OracleChunkEngine:
    """CPU stand-in for GrapeEngine's slice-chunk interface (tests of parallel.py): the same packed
    products and boundary values, restated with numpy on the eigh propagators (qoc.py:128-134)."""

    def __init__(self, system):
        import torch

        self.system = system
        self.torch_device = torch.device("cpu")

    def close(self):
        pass

    def _unpack(self, flat):
        out, o = [], 0
        for blk in self.system.blocks:
            d = blk.dim
            out.append(flat[o:o + d * d].reshape(d, d))
            o += d * d
        return out

    def objective_t(self, u_t):
        import torch

        F, g, _ = objective(self.system, u_t.numpy())
        return torch.tensor([F], dtype=torch.float64), torch.from_numpy(g)

    def chunk_forward_t(self, u_t):
        import torch

        u = u_t.numpy()
        parts = []
        for blk in self.system.blocks:
            x = np.eye(blk.dim, dtype=np.complex128)
            for j in range(u.shape[1]):
                uj, _ = expm_hermitian(hamiltonian(blk.h0, blk.hk, u[:, j]), self.system.dt)
                x = uj @ x
            parts.append(x.reshape(-1))
        return torch.from_numpy(np.concatenate(parts).view(np.float64).copy())

    def chunk_backward_t(self, u_t, gathered, n_chunks, chunk):
        import torch

        u = u_t.numpy()
        prods = [self._unpack(gathered[i].numpy().view(np.complex128)) for i in range(n_chunks)]
        w = self.system.block_weights()
        F = 0.0
        grad = np.zeros(np.shape(u))
        for b, blk in enumerate(self.system.blocks):
            left = np.eye(blk.dim, dtype=np.complex128)
            for i in range(chunk):
                left = prods[i][b] @ left
            right = np.eye(blk.dim, dtype=np.complex128)
            for i in range(chunk + 1, n_chunks):
                right = prods[i][b] @ right
            tgt = np.asarray(self.system.targets[b], dtype=np.complex128)
            lam_end = right.conj().T @ tgt
            if self.system.objective == "gate":
                tau = np.vdot(lam_end, prods[chunk][b] @ left)
                _, dt = gate_dtau(lam_end, u, blk.h0, blk.hk, self.system.dt, x0=left, lam_end=lam_end)
            else:
                psi_start = left @ np.asarray(self.system.initial[b], dtype=np.complex128)
                tau = np.vdot(lam_end, prods[chunk][b] @ psi_start)
                _, dt = state_dtau(psi_start, lam_end, u, blk.h0, blk.hk, self.system.dt)
            F += w[b] * abs(tau) ** 2
            grad += 2.0 * w[b] * np.real(np.conj(tau) * dt)
        return torch.tensor([F], dtype=torch.float64), torch.from_numpy(grad)
