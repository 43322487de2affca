"""Round-2 golden fixtures: BASELINE-size parity cases and reference-pinned basis columns.

Usage (build container only; /root/reference must exist):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fixtures_r02.py [part ...]

parts: adjoint armijo cfg4 cfg2 cfg3 cfg1 (default: all).  Each part writes its own
``tests/golden/r02_<part>.npz`` so the expensive ones can be regenerated alone.

What comes from where:

* ``adjoint``  -- REFERENCE: ``adjoint.build_full_adjoint(n, "dn")`` columns for n = 8, 10
  (the block/column indexing contract, adjoint.py:198-220 + groups.py:298-307), stored as
  CSC arrays.
* ``armijo``   -- REFERENCE: ``qoc.optimize`` (qoc.py:171-219) on the reference's own
  nearest-neighbour n = 4 model, full and first-block-d backends: objective trace and final
  schedule, plus the matrices / states / initial schedule the GPU run needs.
* ``cfg4``     -- REFERENCE: ``qoc.gradient`` (qoc.py:137-168) through a duck-typed backend on
  the repo's cfg 4 systems: the n = 12 A1 block (d = 224) at the full N_t = 200, and the
  unsymmetrised 4096-dim space at N_t = 2 (two eigh of 4096 per slice).
* ``cfg2``, ``cfg3``, ``cfg1`` -- ORACLE (oracle/grape_oracle.py, itself pinned to the
  reference in tests/test_oracle.py): the gate-fidelity objective has no gradient in the
  reference (SURVEY 8c gap G2).  cfg 2 at its full N_t = 500; cfg 3 with all 16 D_14 blocks
  at N_t = 4 (dt = 0.02 as the config); cfg 1: 16 sampled rows of the 4096-seed bench batch
  (rows 0 and 4095 included) at the full N_t = 1000.

Inputs are rebuilt on the GPU box by ``systems.config`` with the same seeds (numpy's
default_rng is platform independent); each fixture stores an input checksum the tests
compare first.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

CFG1_ROWS = [0, 1, 2, 3, 127, 128, 511, 1024, 2047, 2048, 3000, 4000, 4093, 4094, 4095, 777]


def checksum(*arrays) -> np.ndarray:
    """Order-sensitive fingerprint of the inputs (sum and weighted sum of every array)."""
    out = []
    for a in arrays:
        a = np.asarray(a).astype(np.complex128).ravel()
        w = np.arange(1, a.size + 1, dtype=np.float64)
        out += [a.sum(), (w * a).sum() / a.size]
    return np.array(out)


def part_adjoint():
    from symqoc import adjoint

    g = {}
    for n in (8, 10):
        a = adjoint.build_full_adjoint(n, "dn")
        m = a.matrix.sparse().tocsc()
        m.eliminate_zeros()
        g[f"dn{n}_sizes"] = np.array(a.blocks.sizes)
        assert np.abs(m.data.imag).max() == 0.0  # the D_n basis is real
        g[f"dn{n}_data"] = m.data.real.copy()
        g[f"dn{n}_indices"] = m.indices.astype(np.int32)
        g[f"dn{n}_indptr"] = m.indptr.astype(np.int32)
    return g


def part_armijo():
    from symqoc import model, qoc
    from symqoc.propagate import Backend, TimeGrid

    g = {}
    cfg = model.nearest_neighbor_config(4)
    grid = TimeGrid(10.0, 30)
    for kind in ("full", "first-block-d"):
        prob = qoc.QocProblem(cfg, grid, backend=kind, max_iterations=25)
        res = qoc.optimize(prob)
        be = Backend(cfg, kind)
        s0 = qoc.initial_schedule(prob)
        key = "armijo_" + kind.replace("-", "_")
        g.update({f"{key}_{k}": v for k, v in dict(
            h0=be.h0, hx=be.hx, hy=be.hy, psi0=be.basis_state("all-up"), psif=be.basis_state("all-down"),
            bx0=s0.bx, by0=s0.by, tau=grid.tau, trace=np.array(res.objective_trace),
            bx=res.schedule.bx, by=res.schedule.by, converged=res.converged).items()})
    return g


class Duck:
    def __init__(self, h0, hx, hy):
        self.h0, self.hx, self.hy = h0, hx, hy
        self.dim = h0.shape[0]

    def hamiltonian(self, bx, by):
        return self.h0 + bx * self.hx + by * self.hy


def part_cfg4():
    from symqoc import qoc

    from paper_2309_05884_b200 import systems

    g = {}
    for tag, n_sl, full in (("a1", 200, False), ("full", 2, True)):
        s = systems.config(4, n_slices=n_sl, full=full)
        u = s.controls(11)
        blk = s.blocks[0]
        t0 = time.time()
        gx, gy, p = qoc.gradient(s.initial[0], s.targets[0], u[0], u[1], Duck(blk.h0, *blk.hk), s.dt)
        print(f"cfg4 {tag}: reference qoc.gradient {time.time() - t0:.1f} s", flush=True)
        g[f"cfg4_{tag}_F"] = p
        g[f"cfg4_{tag}_grad"] = np.stack([gx, gy])
        g[f"cfg4_{tag}_check"] = checksum(u, s.targets[0], s.initial[0], blk.h0[:64, :64])
    return g


def _oracle_gate(cfg, n_slices, rows=None, seed=11):
    from oracle import grape_oracle

    from paper_2309_05884_b200 import systems

    s = systems.config(cfg, n_slices=n_slices) if n_slices else systems.config(cfg)
    g = {}
    if rows is None:
        u = s.controls(seed)
        t0 = time.time()
        F, grad, per_block = grape_oracle.objective(s, u)
        print(f"cfg{cfg}: oracle {time.time() - t0:.1f} s", flush=True)
        g[f"cfg{cfg}_F"] = F
        g[f"cfg{cfg}_grad"] = grad
        g[f"cfg{cfg}_per_block"] = per_block
        g[f"cfg{cfg}_check"] = checksum(u, *[t[:8, :8] for t in s.targets], *[b.h0[:8, :8] for b in s.blocks])
    else:
        ub = s.controls(0, batch=4096)  # bench.py rank 0 batch (seed0 = 0)
        Fs, grads = [], []
        t0 = time.time()
        for r in rows:
            F, grad, _ = grape_oracle.objective(s, ub[r])
            Fs.append(F)
            grads.append(grad)
        print(f"cfg{cfg}: oracle {len(rows)} rows {time.time() - t0:.1f} s", flush=True)
        g[f"cfg{cfg}_rows"] = np.array(rows)
        g[f"cfg{cfg}_F"] = np.array(Fs)
        g[f"cfg{cfg}_grad"] = np.array(grads)
        g[f"cfg{cfg}_check"] = checksum(ub[rows], *[t for t in s.targets], *[b.h0 for b in s.blocks])
    return g


def part_cfg2():
    return _oracle_gate(2, None)


def part_cfg3():
    return _oracle_gate(3, 4)


def part_cfg1():
    return _oracle_gate(1, None, rows=CFG1_ROWS)


PARTS = {"adjoint": part_adjoint, "armijo": part_armijo, "cfg4": part_cfg4, "cfg2": part_cfg2,
         "cfg3": part_cfg3, "cfg1": part_cfg1}


def main(names):
    for name in names or list(PARTS):
        t0 = time.time()
        g = PARTS[name]()
        path = os.path.join(HERE, f"r02_{name}.npz")
        np.savez_compressed(path, **g)
        print(f"wrote {path}: {len(g)} arrays in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
