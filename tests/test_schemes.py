"""The shipped propagator-scheme coefficients (csrc/schemes.h) reproduce the Taylor series of
exp through their degree, and evaluate exp(A) to double precision at their theta."""

import math
import os
import re

import numpy as np
import pytest
import scipy.linalg

HDR = os.path.join(os.path.dirname(__file__), "..", "paper_2309_05884_b200", "csrc", "schemes.h")


def constants():
    c = {}
    for m in re.finditer(r"#define SQOC_(S[45]_\w+)\s+(\S+)", open(HDR).read()):
        c[m.group(1)] = float(m.group(2))
    return c


def pmul(p, q):
    return np.convolve(p, q)


def padd(p, q):
    n = max(len(p), len(q))
    return np.pad(p, (0, n - len(p))) + np.pad(q, (0, n - len(q)))


def s4_poly(c):
    Z = np.array([c["S4_Z0"], c["S4_Z1"], c["S4_Z2"], c["S4_Z3"], c["S4_X4"], c["S4_X5"], c["S4_X6"]])
    b = np.array([c["S4_B0"], c["S4_B1"], c["S4_B2"], c["S4_B3"]])
    cc = np.array([c["S4_C0"], c["S4_C1"], c["S4_C2"], c["S4_C3"]])
    return padd(pmul(padd(Z, b), Z), cc)


def s5_poly(c):
    basis = lambda v: np.array([v[0], v[1], v[2], v[3], 0, 0, v[4]])  # noqa: E731
    P = np.array([0.0, 1.0, c["S5_BE2"], c["S5_BE3"]])
    Q = np.array([0, 0, c["S5_GA2"], c["S5_GA3"], 0, 0, c["S5_GA6"]])
    Z = pmul(P, Q)
    b = basis([c[f"S5_B{k}"] for k in (0, 1, 2, 3, 6)])
    e = basis([c[f"S5_E{k}"] for k in (0, 1, 2, 3, 6)])
    cc = basis([c[f"S5_C{k}"] for k in (0, 1, 2, 3, 6)])
    return padd(pmul(padd(Z, b), padd(Z, e)), cc)


@pytest.mark.parametrize("name,degree", [("s4", 12), ("s5", 18)])
def test_scheme_is_taylor(name, degree):
    y = (s4_poly if name == "s4" else s5_poly)(constants())
    assert len(y) == degree + 1  # no terms beyond the degree
    for k in range(degree + 1):
        assert abs(y[k] * math.factorial(k) - 1.0) < 1e-12, (name, k, y[k] * math.factorial(k))


def _apply(name, A, c):
    I = np.eye(len(A))
    A2 = A @ A
    A3 = A2 @ A
    if name == "s4":
        P = c["S4_X6"] * A3 + c["S4_X4"] * A + c["S4_X5"] * A2
        Z = P @ A3 + c["S4_Z0"] * I + c["S4_Z1"] * A + c["S4_Z2"] * A2 + c["S4_Z3"] * A3
        W = Z + c["S4_B0"] * I + c["S4_B1"] * A + c["S4_B2"] * A2 + c["S4_B3"] * A3
        return W @ Z + c["S4_C0"] * I + c["S4_C1"] * A + c["S4_C2"] * A2 + c["S4_C3"] * A3
    A6 = A3 @ A3
    basis = [I, A, A2, A3, A6]
    lin = lambda p: sum(c[f"S5_{p}{k}"] * M for k, M in zip((0, 1, 2, 3, 6), basis))  # noqa: E731
    P = A + c["S5_BE2"] * A2 + c["S5_BE3"] * A3
    Q = c["S5_GA2"] * A2 + c["S5_GA3"] * A3 + c["S5_GA6"] * A6
    Z = P @ Q
    return (Z + lin("B")) @ (Z + lin("E")) + lin("C")


@pytest.mark.parametrize("name,theta", [("s4", 0.33), ("s5", 1.10)])
def test_scheme_accuracy_at_theta(name, theta):
    rng = np.random.default_rng(7)
    c = constants()
    for d in (5, 13, 40):
        H = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        H = (H + H.conj().T) / 2
        A = -1j * H
        A *= theta / np.abs(A).sum(1).max()
        err = np.abs(_apply(name, A, c) - scipy.linalg.expm(A)).max()
        assert err < 2e-15, (name, d, err)
