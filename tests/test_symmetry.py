"""Host block bases reproduce the reference's block indexing and matrices."""

import numpy as np
import pytest

from paper_2309_05884_b200 import pauli, symmetry, systems


@pytest.mark.parametrize("n", [6, 8, 10])
def test_dn_block_sizes_match_reference(golden, n):
    assert tuple(b.dim for b in symmetry.dn_full_basis(n)) == tuple(golden[f"dn{n}_sizes"])


def test_bracelet_dims_match_reference(golden):
    dims = [symmetry.bracelet_block(n).dim for n in range(3, 15)]
    assert dims == list(golden["bracelet_dims"])
    # Table 1 of the paper
    assert dims == [4, 6, 8, 13, 18, 30, 46, 78, 126, 224, 380, 687]


def test_dn6_generators_match_reference(golden):
    sysm = systems.gate_ring(6, 10.0, 10)
    for b, blk in enumerate(sysm.blocks):
        for name, m in zip(("h0", "hx", "hy"), (blk.h0, *blk.hk)):
            np.testing.assert_allclose(m, golden[f"dn6_b{b}_{name}"], atol=1e-13)


def test_sn12_sector_generators_match_reference(golden):
    sysm = systems.gate_all_to_all(12, 10.0, 10)
    assert [b.dim for b in sysm.blocks] == [13, 11, 9, 7, 5, 3, 1]
    for blk in sysm.blocks:
        d = blk.dim
        for name, m in zip(("h0", "hx", "hy"), (blk.h0, *blk.hk)):
            np.testing.assert_allclose(m, golden[f"sn12_d{d}_{name}"], atol=1e-12)


def test_bracelet_block_is_dn_a1_block():
    a1 = symmetry.dn_full_basis(8)[0]
    br = symmetry.bracelet_block(8)
    np.testing.assert_allclose(a1.columns.toarray(), br.columns.toarray(), atol=1e-15)


@pytest.mark.parametrize("n", [5, 6, 7])
def test_dn_basis_block_diagonalises_heisenberg_and_controls(n):
    blocks = symmetry.dn_full_basis(n)
    a = np.hstack([b.columns.toarray() for b in blocks])
    np.testing.assert_allclose(a.T @ a, np.eye(1 << n), atol=1e-12)
    ops = [systems.ring_heisenberg(n), *systems.global_controls(n)]
    mask = np.ones((1 << n, 1 << n), dtype=bool)
    s = 0
    for b in blocks:
        mask[s:s + b.dim, s:s + b.dim] = False
        s += b.dim
    for op in ops:
        m = a.T @ pauli.realize(op).toarray() @ a
        assert np.abs(m[mask]).max() <= 1e-12


def test_dn14_block_sizes():
    """n=14 is refused by the reference (adjoint.py:231-232); sizes from the character formula."""
    sizes = [b.dim for b in symmetry.dn_full_basis(14)]
    assert sizes == [687, 495, 549, 613] + [1161, 1161, 1179, 1179] * 3


def test_pauli_term_encoding_for_gpu_compression():
    """gpu_basis.pauli_terms reproduces pauli.realize (CPU check of the GPU compression input)."""
    import numpy as np

    from paper_2309_05884_b200 import gpu_basis, pauli, systems

    n = 5
    for op in (systems.ring_heisenberg(n), *systems.global_controls(n),
               pauli.PauliTermSum(n, [pauli.PauliString(n, "XYZIY", 0.7), pauli.PauliString(n, "YYIZX", -1.3)])):
        flip, sign, coef = gpu_basis.pauli_terms(op)
        dense = np.zeros((1 << n, 1 << n), dtype=np.complex128)
        for f, sg, cr, ci in zip(flip, sign, coef[0::2], coef[1::2]):
            for x in range(1 << n):
                par = bin(x & int(sg)).count("1") & 1
                dense[x ^ int(f), x] += (cr + 1j * ci) * (-1.0 if par else 1.0)
        assert np.abs(dense - pauli.realize(op).toarray()).max() <= 1e-15


def _reference_adjoint(n):
    """Reference ``build_full_adjoint(n, 'dn')`` columns (tests/golden/make_fixtures_r02.py)."""
    import os

    import scipy.sparse as sp

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "r02_adjoint.npz"))
    dim = 1 << n
    m = sp.csc_matrix((z[f"dn{n}_data"], z[f"dn{n}_indices"], z[f"dn{n}_indptr"]), shape=(dim, dim))
    return m.toarray(), list(z[f"dn{n}_sizes"])


@pytest.mark.parametrize("n", [8, 10])
def test_dn_columns_match_reference(n):
    """Block order AND column order/values of the full D_n basis equal the reference's
    (adjoint.py:198-220; the indexing contract), not just the sizes."""
    ref, sizes = _reference_adjoint(n)
    blocks = symmetry.dn_full_basis(n)
    assert [b.dim for b in blocks] == sizes
    ours = np.hstack([b.columns.toarray() for b in blocks])
    assert np.abs(ours - ref).max() <= 1e-14
    # the generating Fock index of each column is its smallest-(weight, index) support state
    s = 0
    for b in blocks:
        for c, key in enumerate(b.keys):
            assert ref[key[1], s + c] != 0.0
        s += b.dim


def test_sn_multiplets_are_spin_eigenvectors():
    """sn_multiplet columns: orthonormal, S_z = M, S^2 = J(J+1) (n = 8, every J)."""
    n = 8
    sz = np.array([(n - 2 * bin(x).count("1")) / 2 for x in range(1 << n)])
    hx, hy = (pauli.realize(o).toarray() for o in systems.global_controls(n))
    sx, sy = hx / 2, hy / 2
    szm = np.diag(sz)
    s2 = sx @ sx + sy @ sy + szm @ szm
    for two_j in range(n, -1, -2):
        cols = symmetry.sn_multiplet(n, two_j)
        assert np.abs(cols.T @ cols - np.eye(two_j + 1)).max() <= 1e-13
        j = two_j / 2
        for k in range(two_j + 1):
            m = j - k
            v = cols[:, k]
            assert np.abs(sz * v - m * v).max() <= 1e-13
            assert np.abs(s2 @ v - j * (j + 1) * v).max() <= 1e-12
