"""On-GPU D_n basis construction and compression against the host restatement
and the reference.

The host restatement (symmetry.dn_full_basis) is pinned to the reference's own
adjoint._dn_full_projected: block sizes at n = 6, 8, 10 and every column at n = 8, 10
(tests/test_symmetry.py, fixture tests/golden/r02_adjoint.npz).  Here the GPU builder must
give the same blocks in the same order with the same column order (bit-exact keys) and the
same column values / compressed generators to rounding -- and, at n = 8, 10, the reference's
columns directly.
"""

import time

import numpy as np
import pytest

from paper_2309_05884_b200 import gpu_basis, systems, symmetry
from paper_2309_05884_b200.engine import GrapeEngine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8, 10, 12])
def test_gpu_basis_matches_host_restatement(n):
    host = symmetry.dn_full_basis(n)
    gb = gpu_basis.GpuDnBasis(n)
    try:
        dev = gb.blocks()
        assert [b.label for b in dev] == [b.label for b in host]
        assert [b.dim for b in dev] == [b.dim for b in host]
        for bd, bh in zip(dev, host):
            assert bd.keys == bh.keys  # column order, bit-exact
            diff = abs(bd.columns - bh.columns)
            assert (diff.max() if diff.nnz else 0.0) <= 1e-14
            # orthonormal columns
            g = (bd.columns.T @ bd.columns).toarray()
            assert np.abs(g - np.eye(bd.dim)).max() <= 1e-13
        for op in (systems.ring_heisenberg(n), *systems.global_controls(n)):
            from paper_2309_05884_b200 import pauli

            full = pauli.realize(op)
            mats = gb.compress(op)
            for m, bh in zip(mats, host):
                ref = bh.compress(full)
                assert np.abs(m - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    finally:
        gb.close()


@pytest.mark.parametrize("n", [8, 10])
def test_gpu_basis_columns_match_reference(n):
    """GPU-built columns against the reference's build_full_adjoint(n, 'dn') (adjoint.py:198-220)."""
    import os

    import scipy.sparse as sp

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "r02_adjoint.npz"))
    dim = 1 << n
    ref = sp.csc_matrix((z[f"dn{n}_data"], z[f"dn{n}_indices"], z[f"dn{n}_indptr"]), shape=(dim, dim)).toarray()
    gb = gpu_basis.GpuDnBasis(n)
    try:
        dev = gb.blocks()
        assert [b.dim for b in dev] == list(z[f"dn{n}_sizes"])
        ours = np.hstack([b.columns.toarray() for b in dev])
        assert np.abs(ours - ref).max() <= 1e-14
    finally:
        gb.close()


def test_gpu_basis_n14_block_sizes_and_speed():
    t0 = time.perf_counter()
    gb = gpu_basis.GpuDnBasis(14)
    try:
        mats = [gb.compress(t) for t in (systems.ring_heisenberg(14), *systems.global_controls(14))]
        dt = time.perf_counter() - t0
        # 687, 495, 549, 613, then (1161, 1161, 1179, 1179) x 3
        assert gb.dims == [687, 495, 549, 613] + [1161, 1161, 1179, 1179] * 3
        assert gb.labels()[:4] == ["A1", "A2", "B1", "B2"]
        for m in mats:  # Hermitian (H0, ΣX) and Hermitian (ΣY) generators
            for h in m:
                assert np.abs(h - h.conj().T).max() <= 1e-12
        assert dt < 15.0  # host restatement: ~21 s for the basis alone
    finally:
        gb.close()


def test_gpu_built_system_gives_same_objective():
    s_host = systems.gate_ring(8, 10.0, 20)
    s_gpu = systems.gate_ring(8, 10.0, 20, builder="gpu")
    u = s_host.controls(3, batch=2)
    e1 = GrapeEngine(s_host, max_batch=2)
    e2 = GrapeEngine(s_gpu, max_batch=2)
    F1, g1 = e1.objective(u)
    F2, g2 = e2.objective(u)
    assert np.abs(np.asarray(F1) - np.asarray(F2)).max() <= 1e-12
    assert np.abs(np.asarray(g1) - np.asarray(g2)).max() <= 1e-10 * np.abs(g1).max()


def test_gpu_basis_odd_n15_against_host_and_n16_completeness():
    """Beyond the reference's n <= 10: n = 15 (odd, no B irreps) matches the host restatement
    column for column; n = 16 (the ABI maximum) spans the 65536-dim space with orthonormal columns."""
    host = symmetry.dn_full_basis(15)
    gb = gpu_basis.GpuDnBasis(15)
    try:
        dev = gb.blocks()
        assert [b.label for b in dev] == [b.label for b in host]
        assert [b.keys for b in dev] == [b.keys for b in host]
        for bd, bh in zip(dev, host):
            diff = abs(bd.columns - bh.columns)
            assert (diff.max() if diff.nnz else 0.0) <= 1e-14
    finally:
        gb.close()
    gb = gpu_basis.GpuDnBasis(16)
    try:
        assert sum(gb.dims) == 1 << 16
        dev = gb.blocks()
        for b in dev[:4] + dev[-2:]:
            g = (b.columns.T @ b.columns).toarray()
            assert np.abs(g - np.eye(b.dim)).max() <= 1e-13
    finally:
        gb.close()
