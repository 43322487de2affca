"""The five BASELINE systems as block generators + seeded synthetic inputs.

Models (BASELINE.json ``configs``; SURVEY.md section 8c gap G1): the reference's
``model.py:59-92`` only builds Ising rings with 1/2 and 1/4 factors, so the
Heisenberg terms are assembled here directly from Pauli strings with the
reference's conventions (``pauli.py:28-221``):

* ring:        H0 = J sum_i (X_i X_{i+1} + Y_i Y_{i+1} + Z_i Z_{i+1}) + h sum_i Z_i, periodic
* all-to-all:  H0 = (J/n) sum_{i<j} (X_i X_j + Y_i Y_j + Z_i Z_j) + h sum_i Z_i
* controls:    H1 = sum_i X_i,  H2 = sum_i Y_i  (coefficient 1.0)

with J = 1, h = 0.5.  Random inputs follow the reference's convention
``numpy.random.default_rng(seed)`` (``qoc.py:103``, gap G6): controls
u ~ Uniform[-1, 1] with u[0] -> H1 (the reference's ``bx``) and u[1] -> H2
(``by``); Haar states are normalised complex Gaussians; Haar unitaries are QR of
a complex Gaussian with the R-diagonal phase fixed.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import pauli, symmetry

J_COUPLING = 1.0
H_BIAS = 0.5


def ring_heisenberg(n: int, j: float = J_COUPLING, h: float = H_BIAS) -> pauli.PauliTermSum:
    terms = []
    for i in range(1, n + 1):
        k = i % n + 1
        for letter in "XYZ":
            terms.append(pauli.pair(n, i, k, letter, j))
    terms += [pauli.single_site(n, i, "Z", h) for i in range(1, n + 1)]
    return pauli.PauliTermSum(n, terms)


def all_to_all_heisenberg(n: int, j: float = J_COUPLING, h: float = H_BIAS) -> pauli.PauliTermSum:
    terms = []
    for a in range(1, n + 1):
        for b in range(a + 1, n + 1):
            for letter in "XYZ":
                terms.append(pauli.pair(n, a, b, letter, j / n))
    terms += [pauli.single_site(n, i, "Z", h) for i in range(1, n + 1)]
    return pauli.PauliTermSum(n, terms)


def global_controls(n: int):
    hx = pauli.PauliTermSum(n, [pauli.single_site(n, i, "X") for i in range(1, n + 1)])
    hy = pauli.PauliTermSum(n, [pauli.single_site(n, i, "Y") for i in range(1, n + 1)])
    return hx, hy


def haar_state(rng: np.random.Generator, d: int) -> np.ndarray:
    psi = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    return psi / np.linalg.norm(psi)


def haar_unitary(rng: np.random.Generator, d: int) -> np.ndarray:
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


@dataclass
class Block:
    """Dense generators of one symmetry block (complex128, row-major)."""

    label: str
    h0: np.ndarray
    hk: list  # control generators, same shape as h0
    basis: symmetry.BlockBasis | None = None

    @property
    def dim(self) -> int:
        return self.h0.shape[0]


@dataclass
class GrapeSystem:
    """One fidelity+gradient workload: blocks, objective, time grid, targets."""

    name: str
    n_qubits: int
    blocks: list
    objective: str  # 'gate' | 'state'
    T: float
    n_slices: int
    targets: list  # gate: V_b (d,d); state: psi_f (d,)
    initial: list = field(default_factory=list)  # state: psi_0 (d,) per block
    weights: np.ndarray | None = None

    @property
    def dt(self) -> float:
        # an empty grid has no slices to scale; any positive dt is equivalent (TimeGrid, propagate.py:36-38)
        return self.T / self.n_slices if self.n_slices else 1.0

    @property
    def n_controls(self) -> int:
        return len(self.blocks[0].hk)

    def block_weights(self) -> np.ndarray:
        """F = sum_b w_b |tau_b|^2: mean of per-block gate fidelities, or |<psi_f|psi_N>|^2."""
        if self.weights is not None:
            return np.asarray(self.weights, dtype=np.float64)
        if self.objective == "gate":
            nb = len(self.blocks)
            return np.array([1.0 / (nb * b.dim**2) for b in self.blocks])
        return np.ones(len(self.blocks))

    def controls(self, seed: int, batch: int | None = None) -> np.ndarray:
        """u ~ Uniform[-1, 1], shape (K, N) or (batch, K, N)."""
        rng = np.random.default_rng(seed)
        shape = (self.n_controls, self.n_slices) if batch is None else (batch, self.n_controls, self.n_slices)
        return rng.uniform(-1.0, 1.0, shape)

    def flops_per_eval(self, g: int | None = None) -> float:
        """Algorithmic FLOPs of one evaluation: 8 N G sum_b d_b^3."""
        if g is None:
            g = 22 if self.objective == "gate" else 8
        return 8.0 * self.n_slices * g * sum(float(b.dim) ** 3 for b in self.blocks)


def hermitian_part(m: np.ndarray) -> np.ndarray:
    """(M + M^dagger)/2: removes the ~1e-16 asymmetry the sparse triple product leaves."""
    return 0.5 * (m + m.conj().T)


def _blocks_from_basis(bases, h0, hk):
    return [
        Block(b.label, hermitian_part(b.compress(h0)), [hermitian_part(b.compress(h)) for h in hk], b)
        for b in bases
    ]


def _operators(n, model):
    h0 = pauli.realize(ring_heisenberg(n) if model == "ring" else all_to_all_heisenberg(n))
    hx, hy = global_controls(n)
    return h0, [pauli.realize(hx), pauli.realize(hy)]


def state_transfer_ring(n: int, T: float, n_slices: int, seed: int = 0, full: bool = False) -> GrapeSystem:
    """|0..0> -> Haar state in the A1 (bracelet) block; block path or unsymmetrised 2^n."""
    h0, hk = _operators(n, "ring")
    a1 = symmetry.bracelet_block(n)
    rng = np.random.default_rng((seed, 0x7A6))
    phi_f = haar_state(rng, a1.dim)
    if full:
        import scipy.sparse as sp

        blk = Block("full", np.asarray(h0.todense()), [np.asarray(h.todense()) for h in hk], None)
        psi0 = np.zeros(1 << n, dtype=np.complex128)
        psi0[0] = 1.0
        psif = a1.from_block(phi_f).astype(np.complex128)
        return GrapeSystem(f"ring{n}-full", n, [blk], "state", T, n_slices, [psif], [psi0])
    blk = _blocks_from_basis([a1], h0, hk)[0]
    psi0 = np.zeros(a1.dim, dtype=np.complex128)
    psi0[0] = 1.0  # |0...0> is bracelet column 0 (propagate.py:107-115)
    return GrapeSystem(f"ring{n}-A1", n, [blk], "state", T, n_slices, [phi_f], [psi0])


def gate_ring(n: int, T: float, n_slices: int, seed: int = 0, builder: str = "host") -> GrapeSystem:
    """D_n-blocked ring, gate fidelity per block.  ``builder="gpu"`` builds the basis and the
    compressed generators on the GPU (gpu_basis.py); same blocks, same order."""
    if builder == "gpu":
        from . import gpu_basis

        gb = gpu_basis.GpuDnBasis(n)
        try:
            bases = gb.blocks()
            mats = [gb.compress(t) for t in (ring_heisenberg(n), *global_controls(n))]
        finally:
            gb.close()
        blocks = [
            Block(b.label, hermitian_part(mats[0][i]), [hermitian_part(mats[1][i]), hermitian_part(mats[2][i])], b)
            for i, b in enumerate(bases)
        ]
    elif builder == "host":
        h0, hk = _operators(n, "ring")
        blocks = _blocks_from_basis(symmetry.dn_full_basis(n), h0, hk)
    else:
        raise ValueError(f"unknown basis builder {builder!r}")
    rng = np.random.default_rng((seed, 0x6A7E))
    targets = [haar_unitary(rng, b.dim) for b in blocks]
    return GrapeSystem(f"ring{n}-Dn", n, blocks, "gate", T, n_slices, targets)


def gate_all_to_all(n: int, T: float, n_slices: int, seed: int = 0) -> GrapeSystem:
    h0, hk = _operators(n, "all")
    blocks = _blocks_from_basis(symmetry.sn_sector_blocks(n), h0, hk)
    rng = np.random.default_rng((seed, 0x6A7E))
    targets = [haar_unitary(rng, b.dim) for b in blocks]
    return GrapeSystem(f"a2a{n}-Sn", n, blocks, "gate", T, n_slices, targets)


def config(index: int, seed: int = 0, **overrides) -> GrapeSystem:
    """BASELINE.json configs[index].

    ``n_slices`` may be overridden for short runs; dt stays the config's dt
    (T scales with N) unless ``T`` is given too.
    """
    base_n = {0: 100, 1: 1000, 2: 500, 3: 500, 4: 200}[index]
    n_sl = overrides.get("n_slices", base_n)
    T = overrides.get("T", 10.0 * n_sl / base_n)
    if index == 0:
        return state_transfer_ring(overrides.get("n", 6), T, n_sl, seed)
    if index == 1:
        return gate_all_to_all(overrides.get("n", 12), T, n_sl, seed)
    if index == 2:
        return gate_ring(overrides.get("n", 10), T, n_sl, seed, builder=overrides.get("builder", "host"))
    if index == 3:
        return gate_ring(overrides.get("n", 14), T, n_sl, seed, builder=overrides.get("builder", "host"))
    if index == 4:
        return state_transfer_ring(overrides.get("n", 12), T, n_sl, seed, full=overrides.get("full", True))
    raise ValueError(f"no config {index}")


CONFIG_BATCH = {0: 1, 1: 4096, 2: 1, 3: 1, 4: 1}
