"""Generate golden vectors by running the REFERENCE package (build container only).

Usage:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here is an output of ``symqoc`` itself (its Pauli realiser,
basis builders, ``qoc.gradient``, ``propagate.expm_hermitian`` and
``propagate.unitary_fidelity``); the models the BASELINE configs need but the
reference's ``model.py`` lacks (Heisenberg ring / all-to-all) are assembled from
the reference's own ``PauliString``/``PauliTermSum``.  The npz files are
committed so that tests on the GPU box (where /root/reference does not exist)
can pin both the oracle and the CUDA path to the reference.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from symqoc import adjoint, model, qoc  # noqa: E402
from symqoc.pauli import PauliString, PauliTermSum, realize  # noqa: E402
from symqoc.propagate import Backend, TimeGrid, expm_hermitian, unitary_fidelity  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def letters(n, sites, ch):
    return "".join(ch if k in sites else "I" for k in range(1, n + 1))


def ring(n, j=1.0, h=0.5):
    t = [PauliString(n, letters(n, (i, i % n + 1), c), j) for i in range(1, n + 1) for c in "XYZ"]
    t += [PauliString(n, letters(n, (i,), "Z"), h) for i in range(1, n + 1)]
    return PauliTermSum(n, tuple(t))


def all_to_all(n, j=1.0, h=0.5):
    t = [PauliString(n, letters(n, (a, b), c), j / n)
         for a in range(1, n + 1) for b in range(a + 1, n + 1) for c in "XYZ"]
    t += [PauliString(n, letters(n, (i,), "Z"), h) for i in range(1, n + 1)]
    return PauliTermSum(n, tuple(t))


def controls(n):
    hx = PauliTermSum(n, tuple(PauliString(n, letters(n, (i,), "X"), 1.0) for i in range(1, n + 1)))
    hy = PauliTermSum(n, tuple(PauliString(n, letters(n, (i,), "Y"), 1.0) for i in range(1, n + 1)))
    return hx, hy


class DuckBackend:
    """The duck-typed backend qoc.gradient needs (.dim, .hx, .hy, .hamiltonian)."""

    def __init__(self, h0, hx, hy):
        self.h0, self.hx, self.hy = h0, hx, hy
        self.dim = h0.shape[0]

    def hamiltonian(self, bx, by):
        return self.h0 + bx * self.hx + by * self.hy


def full_blocks(n, group, ops):
    a = adjoint.build_full_adjoint(n, group)
    sizes = a.blocks.sizes
    dense = [np.asarray(a.compress(realize(op))) for op in ops]
    out, s = [], 0
    for d in sizes:
        out.append([m[s:s + d, s:s + d] for m in dense])
        s += d
    return sizes, out


def main():
    g = {}
    # 1) reference qoc.gradient on its own Ising model (test_qoc.py:53-81 setup)
    for n in (2, 3):
        cfg = model.ModelConfig(n, 1.0, (0.2,) if n >= 3 else ())
        be = Backend(cfg, "full")
        grid = TimeGrid(8.0, 25)
        rng = np.random.default_rng(n)
        bx = 0.1 * rng.standard_normal(grid.N)
        by = 0.1 * rng.standard_normal(grid.N)
        psi0, psif = be.basis_state("all-up"), be.basis_state("all-down")
        gx, gy, p = qoc.gradient(psi0, psif, bx, by, be, grid.tau)
        g.update({f"ising{n}_{k}": v for k, v in dict(
            h0=be.h0, hx=be.hx, hy=be.hy, psi0=psi0, psif=psif, bx=bx, by=by,
            tau=grid.tau, gx=gx, gy=gy, P=p).items()})
    # 2) block vs full equivalence case (test_qoc.py:84-99)
    cfg = model.nearest_neighbor_config(4)
    grid = TimeGrid(10.0, 30)
    for kind in ("full", "first-block-d"):
        be = Backend(cfg, kind)
        s = qoc.initial_schedule(qoc.QocProblem(cfg, grid, backend=kind))
        psi0, psif = be.basis_state("all-up"), be.basis_state("all-down")
        gx, gy, p = qoc.gradient(psi0, psif, s.bx, s.by, be, grid.tau)
        key = "nn4_" + kind.replace("-", "_")
        g.update({f"{key}_{k}": v for k, v in dict(
            h0=be.h0, hx=be.hx, hy=be.hy, psi0=psi0, psif=psif, bx=s.bx, by=s.by,
            tau=grid.tau, gx=gx, gy=gy, P=p).items()})
    # 3) cfg 0 system built by the reference: n=6 Heisenberg ring, bracelet block, N=100
    n = 6
    blk = adjoint.build_bracelet_first_block(n)
    h0, (hx, hy) = realize(ring(n)), [realize(o) for o in controls(n)]
    be = DuckBackend(blk.compress(h0), blk.compress(hx), blk.compress(hy))
    rng = np.random.default_rng(1234)
    u = rng.uniform(-1.0, 1.0, (2, 100))
    phi = rng.standard_normal(be.dim) + 1j * rng.standard_normal(be.dim)
    phi /= np.linalg.norm(phi)
    psi0 = np.zeros(be.dim, dtype=np.complex128)
    psi0[0] = 1.0
    gx, gy, p = qoc.gradient(psi0, phi, u[0], u[1], be, 0.1)
    g.update({f"cfg0_{k}": v for k, v in dict(
        h0=be.h0, hx=be.hx, hy=be.hy, psi0=psi0, psif=phi, u=u, tau=0.1, gx=gx, gy=gy, P=p).items()})
    # 4) reference block structure of the full adjoints (indexing contract)
    for n in (6, 8, 10):
        g[f"dn{n}_sizes"] = np.array(adjoint.build_full_adjoint(n, "dn").blocks.sizes)
    g["bracelet_dims"] = np.array([adjoint.build_bracelet_first_block(n).ncols for n in range(3, 15)])
    # 5) reference-compressed block generators: D_6 ring (all blocks), S_12 a2a (first multiplet per J)
    sizes, blocks = full_blocks(6, "dn", [ring(6), *controls(6)])
    for b, mats in enumerate(blocks):
        for name, m in zip(("h0", "hx", "hy"), mats):
            g[f"dn6_b{b}_{name}"] = m
    a = adjoint.build_full_adjoint(12, "sn")
    ops = [np.asarray(a.compress(realize(o))) for o in (all_to_all(12), *controls(12))]
    seen, s0 = {}, 0
    for d in a.blocks.sizes:
        if d not in seen:
            seen[d] = [m[s0:s0 + d, s0:s0 + d] for m in ops]
        s0 += d
    for d, mats in seen.items():
        for name, m in zip(("h0", "hx", "hy"), mats):
            g[f"sn12_d{d}_{name}"] = m
    g["sn12_sizes"] = np.array(a.blocks.sizes)
    # 6) gate fidelity pinned through reference primitives on the D_6 blocks:
    #    X_N = prod expm_hermitian(H_j, dt), F_b = unitary_fidelity(V_b, X_N), central FD of F
    rng = np.random.default_rng(99)
    u = rng.uniform(-1.0, 1.0, (2, 20))
    dt = 0.05
    probes = [(0, 0), (1, 7), (0, 13), (1, 19)]
    for b, (bh0, bhx, bhy) in enumerate(blocks):
        d = bh0.shape[0]
        z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2)
        q, r = np.linalg.qr(z)
        v = q * (np.diag(r) / np.abs(np.diag(r)))[None, :]

        def fid(uu):
            x = np.eye(d, dtype=np.complex128)
            for j in range(uu.shape[1]):
                uj, _ = expm_hermitian(bh0 + uu[0, j] * bhx + uu[1, j] * bhy, dt)
                x = uj.dense() @ x
            return unitary_fidelity(v, x)

        fd = []
        for k, j in probes:
            up, um = u.copy(), u.copy()
            up[k, j] += 1e-6
            um[k, j] -= 1e-6
            fd.append((fid(up) - fid(um)) / 2e-6)
        g[f"gate6_b{b}_V"] = v
        g[f"gate6_b{b}_F"] = fid(u)
        g[f"gate6_b{b}_fd"] = np.array(fd)
    g["gate6_u"] = u
    g["gate6_dt"] = dt
    g["gate6_probes"] = np.array(probes)
    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
