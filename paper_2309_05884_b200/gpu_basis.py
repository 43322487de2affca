"""On-GPU D_n symmetry-adapted basis and block compression.

Thin host wrapper over ``sqoc_dn_basis_create`` / ``sqoc_basis_compress``
(``csrc/basis.cu``): the device builds the orbit tables, the projected and
Gram-Schmidt-orthonormalised columns of every D_n block and the compressed
block generators A_b^T H A_b.  The result is the same block list, in the same
order and column order, as :func:`symmetry.dn_full_basis` (the host restatement
of the reference's ``adjoint._dn_full_projected``, ``adjoint.py:198-220``),
which the tests check block by block.  The reference refuses n > 10
(``adjoint.py:231-232``).  n = 14 on the GPU box: basis 0.03 s and three compressed
operators 0.25 s (mostly the 1 GB of dense blocks copied to the host) against 1.9 s + 0.9 s
for the host restatement (``profiles/r01_basis_times.jsonl``).
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib, pauli, symmetry


def pauli_terms(term_sum: pauli.PauliTermSum):
    """(flip, sign, coef) encoding of a Pauli sum for ``sqoc_basis_compress``.

    P e_x = coef (-1)^popcount(x & sign) e_{x ^ flip}: X/Y letters flip, Z/Y letters
    sign, and sigma_y = i (-1)^bit folds i^#Y into the coefficient (``pauli.py:163-187``).
    """
    n = term_sum.n
    flip, sign, coef = [], [], []
    for t in term_sum.terms:
        f = s = 0
        ny = 0
        for site, letter in enumerate(t.letters, start=1):
            bit = 1 << (n - site)
            if letter in "XY":
                f |= bit
            if letter in "ZY":
                s |= bit
            ny += letter == "Y"
        c = t.coefficient * (1j**ny)
        flip.append(f)
        sign.append(s)
        coef += [c.real, c.imag]
    return (np.asarray(flip, dtype=np.int32), np.asarray(sign, dtype=np.int32), np.asarray(coef, dtype=np.float64))


class GpuDnBasis:
    """Full D_n block basis of n spins built on the GPU."""

    def __init__(self, n: int, device: int | None = None):
        if device is None:  # the caller's current CUDA device (one process per GPU under torchrun)
            try:
                import torch

                device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except ImportError:
                device = 0
        self.lib = _lib.load()
        self.n = n
        h = ctypes.c_void_p()
        _lib.check(self.lib.sqoc_dn_basis_create(ctypes.byref(h), device, n), "sqoc_dn_basis_create")
        self.handle = h
        nb = ctypes.c_int()
        _lib.check(self.lib.sqoc_basis_info(self.handle, ctypes.byref(nb), None, None), "sqoc_basis_info")
        dims = np.zeros(nb.value, dtype=np.int32)
        rows = np.zeros(nb.value, dtype=np.int32)
        _lib.check(self.lib.sqoc_basis_info(self.handle, ctypes.byref(nb), dims.ctypes.data, rows.ctypes.data),
                   "sqoc_basis_info")
        self.dims = [int(d) for d in dims]
        self.irrep_rows = [int(r) for r in rows]

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sqoc_basis_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def labels(self):
        """Block labels in the reference's naming (A1, A2, B1, B2, E_k(j=1|2))."""
        names = ["A1", "A2"] + (["B1", "B2"] if self.n % 2 == 0 else [])
        for k in range(1, (self.n - 1) // 2 + 1):
            names += [f"E{k}(j=1)", f"E{k}(j=2)"]
        return [names[r] for r in self.irrep_rows]

    def blocks(self):
        """The block columns as :class:`symmetry.BlockBasis` objects (sparse, real)."""
        out = []
        for b, (d, label) in enumerate(zip(self.dims, self.labels())):
            nnz = ctypes.c_longlong()
            _lib.check(self.lib.sqoc_basis_nnz(self.handle, b, ctypes.byref(nnz)), "sqoc_basis_nnz")
            keys = np.zeros(d, dtype=np.int32)
            counts = np.zeros(d, dtype=np.int32)
            rows = np.zeros(nnz.value, dtype=np.int32)
            vals = np.zeros(nnz.value, dtype=np.float64)
            _lib.check(self.lib.sqoc_basis_columns(self.handle, b, keys.ctypes.data, counts.ctypes.data,
                                                   rows.ctypes.data, vals.ctypes.data), "sqoc_basis_columns")
            cols = np.repeat(np.arange(d), counts)
            mat = sp.csc_matrix((vals, (rows, cols)), shape=(1 << self.n, d))
            out.append(symmetry.BlockBasis(label, mat, [(bin(int(k)).count("1"), int(k)) for k in keys]))
        return out

    def compress(self, term_sum: pauli.PauliTermSum):
        """A_b^T H A_b (complex128, d_b x d_b) for every block, computed on the GPU."""
        flip, sign, coef = pauli_terms(term_sum)
        outs = [np.zeros((d, d), dtype=np.complex128) for d in self.dims]
        ptrs = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        _lib.check(self.lib.sqoc_basis_compress(self.handle, len(flip), flip.ctypes.data, sign.ctypes.data,
                                                coef.ctypes.data, ptrs), "sqoc_basis_compress")
        return outs

