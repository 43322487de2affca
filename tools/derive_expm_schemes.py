"""Derive the coefficients of the product-saving Taylor evaluation schemes used by the kernels.

Both schemes evaluate a polynomial y(A) that agrees with the Taylor series of exp(A) through
degree m, using fewer matrix products than Paterson-Stockmeyer (PS needs 5 products for
degree 12 and 7 for degree 18).  The idea -- write the polynomial as c(A) + (b(A) + Z) Z with
one "square" of an intermediate polynomial Z -- is the published optimized-Taylor approach of
Sastre / Bader, Blanes & Casas; the structure below and the coefficients are derived here,
from scratch, by solving the coefficient-matching equations in 50-digit arithmetic.

  s4 (degree 12, 4 products):  A2 = A A, A3 = A2 A,
                                Z = (x4 A + x5 A2 + x6 A3) A3 + z0 I + z1 A + z2 A2 + z3 A3,
                                y = (Z + b0 I + b1 A + b2 A2 + b3 A3) Z + c0 I + c1 A + c2 A2 + c3 A3
        13 equations (degrees 0..12), 15 unknowns: the two free parameters are chosen to
        minimise the rounding-error proxy |Z|(t) |Z + b|(t) + |c|(t) at t = theta.
  s5 (degree 18, 5 products):  A2, A3, A6 = A3 A3,
                                Z = (x0 I + x1 A + x2 A2 + x3 A3 + x6 A6) A6 + z0 I + z1 A + z2 A2 + z3 A3,
                                y = (Z + b(A)) Z + c(A),   b, c in span{I, A, A2, A3, A6}
        19 equations (degrees 0..18), 19 unknowns; y has extra terms of degree 19..24 whose
        coefficients are reported (they enter the truncation bound).

python tools/derive_expm_schemes.py   -> prints the C constants and the per-scheme theta
(largest ||A|| with truncation + residual-term bound <= 2^-53).
"""
import itertools
import math

import mpmath as mp
import numpy as np

mp.mp.dps = 50
U = mp.mpf(2) ** -53


def polymul(p, q):
    r = [mp.mpf(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        if a == 0:
            continue
        for j, b in enumerate(q):
            r[i + j] += a * b
    return r


def padd(p, q):
    n = max(len(p), len(q))
    return [(p[i] if i < len(p) else 0) + (q[i] if i < len(q) else 0) for i in range(n)]


def absval(p, t):
    return sum(abs(c) * t ** k for k, c in enumerate(p))


def theta_for(extra, m):
    """Largest t with sum_{k>m} |y_k - 1/k!| t^k <= u (y_k = 0 beyond the residual terms)."""
    def bound(t):
        s = mp.mpf(0)
        for k in range(m + 1, 60):
            yk = extra.get(k, 0)
            s += abs(yk - 1 / mp.factorial(k)) * t ** k
        return s
    lo, hi = mp.mpf("0.01"), mp.mpf(4)
    for _ in range(200):
        mid = (lo + hi) / 2
        if bound(mid) <= U:
            lo = mid
        else:
            hi = mid
    return lo


# ----------------------------------------------------------------------------- s4
def s4_solve(z0, z3, sign=1):
    """Given the free parameters (z0 is a pure gauge: it trades against b0 and c; z3 is the real
    one), solve the degree 4..12 equations.  Top-down: z6, z5, z4 from degrees 12..10, then
    s_k = 2 z_k + b_k (k = 3, 2, 1, 0) from degrees 9..6, z2 from degree 5, z1 from degree 4."""
    inv = [1 / mp.factorial(k) for k in range(13)]
    z6 = sign * mp.sqrt(inv[12])
    z5 = inv[11] / (2 * z6)
    z4 = (inv[10] - z5 ** 2) / (2 * z6)
    s3 = (inv[9] - 2 * z4 * z5) / z6
    s2 = (inv[8] - z4 ** 2 - z5 * s3) / z6
    s1 = (inv[7] - z5 * s2 - z4 * s3) / z6
    b3 = s3 - 2 * z3
    s0 = (inv[6] - z5 * s1 - z4 * s2 - z3 * (z3 + b3)) / z6
    # degree 5: s0 z5 + s1 z4 + z2 (2 z3 + b3) + (s2 - 2 z2) z3 = inv5  ->  z2 b3 = inv5 - s0 z5 - s1 z4 - s2 z3
    z2 = (inv[5] - s0 * z5 - s1 * z4 - s2 * z3) / b3
    b2 = s2 - 2 * z2
    # degree 4: s0 z4 + z1 (2 z3 + b3) + (s1 - 2 z1) z3 + z2 (z2 + b2) = inv4
    z1 = (inv[4] - s0 * z4 - s1 * z3 - z2 * (z2 + b2)) / b3
    b1 = s1 - 2 * z1
    b0 = s0 - 2 * z0
    Z = [z0, z1, z2, z3, z4, z5, z6]
    b = [b0, b1, b2, b3]
    y = padd(polymul(Z, Z), polymul(b, Z))
    c = [inv[k] - y[k] for k in range(4)]
    full = padd(y, c)
    err = max(abs(full[k] - inv[k]) for k in range(13))
    assert err < mp.mpf(10) ** -40, err
    return dict(Z=Z, b=b, c=c)


def s4_proxy(s, t):
    W = padd(s["Z"], s["b"])
    return absval(s["Z"], t) * absval(W, t) + absval(s["c"], t)


def derive_s4(theta=mp.mpf("0.33")):
    best = None
    for sign in (1, -1):
        for z2 in np.linspace(-2, 2, 41):
            for z3 in np.linspace(-0.5, 0.5, 101):
                try:
                    s = s4_solve(mp.mpf(z2), mp.mpf(z3), sign)
                except (ZeroDivisionError, ValueError, TypeError):
                    continue
                p = s4_proxy(s, theta)
                if best is None or p < best[0]:
                    best = (p, z2, z3, sign)
    # local refinement
    p, z2, z3, sign = best
    step = 0.01
    z2, z3 = mp.mpf(z2), mp.mpf(z3)
    for _ in range(60):
        improved = False
        for dz2, dz3 in itertools.product((-step, 0, step), repeat=2):
            s = s4_solve(z2 + dz2, z3 + dz3, sign)
            q = s4_proxy(s, theta)
            if q < p:
                p, z2, z3, improved = q, z2 + dz2, z3 + dz3, True
        if not improved:
            step /= 2
    return s4_solve(z2, z3, sign), p


# ----------------------------------------------------------------------------- s5
# y = (Z + b)(Z + e) + c,  Z = (A + be2 A2 + be3 A3)(ga2 A2 + ga3 A3 + ga6 A6),
# b, e, c in span{I, A, A2, A3, A6}.  Z -> Z + p, b -> b - p, e -> e - p leaves y unchanged for p
# in that span, so only Z's degree 4, 5, 7, 8, 9 coefficients (zeta) matter; they determine
# (be2, be3, ga2, ga3, ga6) uniquely.  With s = b + e, y has no terms above degree 18
# (Z^2: 8..18, sZ: 4..15, be: 0..12), so matching degrees 0..18 makes y = T_18 exactly.
# Solve top-down: zeta9, zeta8, zeta7 from degrees 18..16, s6 from 15, zeta5, zeta4 from 14, 13;
# then for given (b6, s0): s3, s2, s1 from 12..10 and b3, b2, b1 from 9..7 (all linear);
# degrees 5 and 4 leave two equations in (b6, s0), solved by Newton from a grid of starts.
BASIS = [0, 1, 2, 3, 6]


def s5_top():
    inv = [1 / mp.factorial(k) for k in range(19)]
    z9 = mp.sqrt(inv[18])
    z8 = inv[17] / (2 * z9)
    z7 = (inv[16] - z8 ** 2) / (2 * z9)
    s6 = (inv[15] - 2 * z7 * z8) / z9
    z5 = (inv[14] - z7 ** 2 - s6 * z8) / (2 * z9)
    z4 = (inv[13] - 2 * z5 * z8 - s6 * z7) / (2 * z9)
    return inv, dict(z4=z4, z5=z5, z7=z7, z8=z8, z9=z9, s6=s6)


def s5_rest(b6, s0, T):
    inv = T["inv"]
    z4, z5, z7, z8, z9, s6 = (T[k] for k in ("z4", "z5", "z7", "z8", "z9", "s6"))
    e6 = s6 - b6
    s3 = (inv[12] - 2 * z4 * z8 - 2 * z5 * z7 - b6 * e6) / z9
    s2 = (inv[11] - 2 * z4 * z7 - s3 * z8 - s6 * z5) / z9
    s1 = (inv[10] - z5 ** 2 - s2 * z8 - s3 * z7 - s6 * z4) / z9
    den = s6 - 2 * b6
    b3 = (inv[9] - 2 * z4 * z5 - s0 * z9 - s1 * z8 - s2 * z7 - b6 * s3) / den
    b2 = (inv[8] - z4 ** 2 - s0 * z8 - s1 * z7 - s3 * z5 - b6 * s2) / den
    b1 = (inv[7] - s0 * z7 - s2 * z5 - s3 * z4 - b6 * s1) / den
    e1, e2, e3 = s1 - b1, s2 - b2, s3 - b3
    r5 = s0 * z5 + s1 * z4 + b2 * e3 + b3 * e2 - inv[5]
    r4 = s0 * z4 + b1 * e3 + b2 * e2 + b3 * e1 - inv[4]
    return (r5, r4), dict(s=[s0, s1, s2, s3, s6], b=[None, b1, b2, b3, b6])


def s5_assemble(b6, s0, T, b0=None):
    """Full coefficient set: B1 = A + be2 A2 + be3 A3, B5 = ga2 A2 + ga3 A3 + ga6 A6, Z = B1 B5,
    y = (Z + bb) (Z + ee) + cc with bb, ee, cc on the basis I, A, A2, A3, A6."""
    inv = T["inv"]
    _, R = s5_rest(b6, s0, T)
    s0, s1, s2, s3, s6 = R["s"]
    _, b1, b2, b3, b6 = R["b"]
    if b0 is None:
        b0 = mp.mpf(0)  # b0 = 0 keeps c0 = 1 (no cancellation in the identity term)
    b = {0: b0, 1: b1, 2: b2, 3: b3, 6: b6}
    e = {0: s0 - b0, 1: s1 - b1, 2: s2 - b2, 3: s3 - b3, 6: s6 - b6}
    z4, z5, z7, z8, z9 = (T[k] for k in ("z4", "z5", "z7", "z8", "z9"))
    ga6 = z7
    be2, be3 = z8 / z7, z9 / z7
    # z4 = ga3 + be2 ga2, z5 = be2 ga3 + be3 ga2
    det = be2 * be2 - be3
    ga2 = (be2 * z4 - z5) / det
    ga3 = z4 - be2 * ga2
    # Z = B1 B5 also carries ga2 A3 + be3 ga3 A6 (gauge p): compensate in b, e
    p = {3: ga2, 6: be3 * ga3}
    for k, v in p.items():
        b[k] -= v
        e[k] -= v
    B1 = [0, 1, be2, be3]
    B5 = [0, 0, ga2, ga3, 0, 0, ga6]
    Z = polymul(B1, B5)
    bb = [b.get(k, 0) for k in range(7)]
    ee = [e.get(k, 0) for k in range(7)]
    y = polymul(padd(Z, bb), padd(Z, ee))
    cc = [0] * 7
    for k in BASIS:
        cc[k] = inv[k] - y[k]
    full = padd(y, cc)
    err = max(abs(full[k] - inv[k]) for k in range(19))
    hi = max([abs(x) for x in full[19:]] + [0])
    return dict(B1=B1, B5=B5, b=bb, e=ee, c=cc, err=err, hi=hi, Z=Z)


def derive_s5():
    inv, T = s5_top()
    T["inv"] = inv
    sols = []
    for b6 in np.linspace(-3, 3, 61):
        for s0 in np.linspace(-20, 20, 81):
            def F(x, y):
                return list(s5_rest(x, y, T)[0])
            try:
                r = mp.findroot(F, (mp.mpf(b6), mp.mpf(s0)), tol=mp.mpf(10) ** -40, maxsteps=80)
            except (ZeroDivisionError, ValueError, TypeError):
                continue
            x, y = r[0], r[1]
            res = s5_rest(x, y, T)[0]
            if max(abs(res[0]), abs(res[1])) > mp.mpf(10) ** -35:
                continue
            if any(abs(x - u[0]) < 1e-12 and abs(y - u[1]) < 1e-12 for u in sols):
                continue
            sols.append((x, y))
    th = theta_for({}, 18)
    out = []
    for x, y in sols:
        S = s5_assemble(x, y, T)
        if S["err"] > mp.mpf(10) ** -35:
            continue
        W1, W2 = padd(S["Z"], S["b"]), padd(S["Z"], S["e"])
        S["proxy"] = absval(W1, th) * absval(W2, th) + absval(S["c"], th)
        S["theta"] = th
        S["b6s0"] = (x, y)
        out.append(S)
    out.sort(key=lambda S: S["proxy"])
    return out


def fmt(x):
    return mp.nstr(x, 17, min_fixed=-3, max_fixed=3)


if __name__ == "__main__":
    s4, p4 = derive_s4()
    th4 = theta_for({}, 12)
    print("// s4: degree 12 in 4 products; theta =", mp.nstr(th4, 6), " proxy =", mp.nstr(p4, 6))
    print("//   Z = z0..z6:", [fmt(x) for x in s4["Z"]])
    print("//   b = b0..b3:", [fmt(x) for x in s4["b"]])
    print("//   c = c0..c3:", [fmt(x) for x in s4["c"]])
    sols = derive_s5()
    print(f"// s5: {len(sols)} real solutions (b0 = 0); theta_18 =", mp.nstr(theta_for({}, 18), 6),
          "-- the kernels use the first (smallest proxy)")
    for S in sols[:4]:
        print("// proxy", mp.nstr(S["proxy"], 6), "err", mp.nstr(S["err"], 3), "hi", mp.nstr(S["hi"], 3))
        print("//   B1 (I A A2 A3):", [fmt(x) for x in S["B1"]])
        print("//   B5 (A2 A3 A6):", [fmt(S["B5"][k]) for k in (2, 3, 6)])
        print("//   b (I A A2 A3 A6):", [fmt(S["b"][k]) for k in BASIS])
        print("//   e (I A A2 A3 A6):", [fmt(S["e"][k]) for k in BASIS])
        print("//   c (I A A2 A3 A6):", [fmt(S["c"][k]) for k in BASIS])
