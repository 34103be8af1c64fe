"""Exact rational polynomial arithmetic (tests only) for closed-form pins of A(alpha), B(alpha).

A_jl = (2j+1)/2 int_{-1}^{2a-1} P_l(xi+2-2a) P_j(xi) dxi,
B_jl = (2j+1)/2 int_{2a-1}^{1}  P_l(xi-2a)   P_j(xi) dxi        (P:259-268 SS II-A)

evaluated symbolically with fractions.Fraction: Legendre polynomials from Bonnet's
recurrence in the monomial basis, exact Taylor shift, exact antiderivative.  With alpha the
exact binary value of a double, the result is the exact real number, so the oracle's
quadrature build must match it to within a few ulp.
"""
from fractions import Fraction
from math import comb


def legendre_poly(n):
    """Monomial coefficients (ascending) of P_n, exact."""
    P = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for j in range(1, n):
        a = [Fraction(0)] + [Fraction(2 * j + 1, j + 1) * c for c in P[j]]
        b = [Fraction(j, j + 1) * c for c in P[j - 1]] + [Fraction(0)] * 2
        P.append([x - y for x, y in zip(a, b)])
    return P[n]


def shift(p, c):
    """Coefficients of p(x + c)."""
    out = [Fraction(0)] * len(p)
    for i, a in enumerate(p):
        for m in range(i + 1):
            out[m] += a * comb(i, m) * c ** (i - m)
    return out


def mul(p, q):
    out = [Fraction(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        for j, b in enumerate(q):
            out[i + j] += a * b
    return out


def integrate(p, lo, hi):
    s = Fraction(0)
    for i, a in enumerate(p):
        s += a * (hi ** (i + 1) - lo ** (i + 1)) / (i + 1)
    return s


def exact_AB(alpha, k):
    a = Fraction(alpha)
    A = [[Fraction(0)] * k for _ in range(k)]
    B = [[Fraction(0)] * k for _ in range(k)]
    for j in range(k):
        Pj = legendre_poly(j)
        for l in range(k):
            Pl = legendre_poly(l)
            A[j][l] = Fraction(2 * j + 1, 2) * integrate(mul(shift(Pl, 2 - 2 * a), Pj), Fraction(-1), 2 * a - 1)
            B[j][l] = Fraction(2 * j + 1, 2) * integrate(mul(shift(Pl, -2 * a), Pj), 2 * a - 1, Fraction(1))
    return A, B
