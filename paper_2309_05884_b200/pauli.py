"""Pauli-string operators realised as sparse 2^n x 2^n matrices (host-side setup).

Mirrors the reference's operator conventions so that every block matrix the GPU
path consumes is the same matrix the reference would build:

* site 1 is the most significant bit of the Fock index, spin-up = bit 0
  (reference ``pkg/src/symqoc/pauli.py:158-160``);
* each Pauli string is a generalised permutation: column x maps to row
  ``x ^ flipmask`` with a phase from the Z/Y letters, sigma_y|up> = i|down>
  (``pauli.py:163-187``);
* term sums are real-weighted (``pauli.py:52-78``) and duplicates are summed
  (``pauli.py:190-221``).

Unlike the reference this module always returns CSR matrices: storage-kind
selection (``pauli.py:81-155``) is a CPU-memory concern that does not reach the
device path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

MAX_QUBITS = 16
_LETTERS = frozenset("IXYZ")


class DimensionError(ValueError):
    """Qubit count or matrix dimension outside the supported range (``pauli.py:24-25``)."""


@dataclass(frozen=True)
class PauliString:
    """One real-weighted tensor-product Pauli string, e.g. ``0.5 * 'IXZI'``."""

    n: int
    letters: str
    coefficient: float = 1.0

    def __post_init__(self):
        if len(self.letters) != self.n:
            raise ValueError(f"letters {self.letters!r} must have length n={self.n}")
        bad = set(self.letters) - _LETTERS
        if bad:
            raise ValueError(f"unknown Pauli letters {sorted(bad)}")


@dataclass(frozen=True)
class PauliTermSum:
    n: int
    terms: tuple = ()

    def __post_init__(self):
        object.__setattr__(self, "terms", tuple(self.terms))
        for t in self.terms:
            if t.n != self.n:
                raise ValueError("all terms must share the same qubit count")

    def __add__(self, other: "PauliTermSum") -> "PauliTermSum":
        if other.n != self.n:
            raise ValueError("qubit counts differ")
        return PauliTermSum(self.n, self.terms + other.terms)


def string_action(term: PauliString):
    """(rows, cols, phases) of one string acting on all 2^n Fock columns."""
    n = term.n
    dim = 1 << n
    cols = np.arange(dim, dtype=np.int64)
    flip = 0
    phase = np.full(dim, term.coefficient, dtype=np.complex128)
    for site, letter in enumerate(term.letters, start=1):
        if letter == "I":
            continue
        shift = n - site
        bit = (cols >> shift) & 1
        if letter == "Z":
            phase *= 1.0 - 2.0 * bit
        elif letter == "X":
            flip |= 1 << shift
        else:  # Y: sigma_y|0> = i|1>, sigma_y|1> = -i|0>
            flip |= 1 << shift
            phase *= 1j - 2j * bit
    return cols ^ flip, cols, phase


def realize(term_sum: PauliTermSum) -> sp.csr_matrix:
    """The 2^n x 2^n complex CSR matrix of a Pauli term sum (duplicates summed)."""
    n = term_sum.n
    if not 1 <= n <= MAX_QUBITS:
        raise DimensionError(f"n={n} outside supported range [1, {MAX_QUBITS}]")
    dim = 1 << n
    if not term_sum.terms:
        return sp.csr_matrix((dim, dim), dtype=np.complex128)
    rows, cols, data = zip(*(string_action(t) for t in term_sum.terms))
    m = sp.coo_matrix(
        (np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
        shape=(dim, dim),
    ).tocsr()
    m.sum_duplicates()
    m.eliminate_zeros()
    return m


def single_site(n: int, site: int, letter: str, coefficient: float = 1.0) -> PauliString:
    letters = "".join(letter if k == site else "I" for k in range(1, n + 1))
    return PauliString(n, letters, coefficient)


def pair(n: int, i: int, j: int, letter: str, coefficient: float = 1.0) -> PauliString:
    letters = "".join(letter if k in (i, j) else "I" for k in range(1, n + 1))
    return PauliString(n, letters, coefficient)
