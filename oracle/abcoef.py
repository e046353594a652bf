"""Adams-Bashforth weights in exact rational arithmetic (ORACLE, test infrastructure).

PAPER.md §3.1 eq:vandermonde and eq:ab_general; §3.2 eq:ext_ab
(P:388-394): for history nodes t_1 < ... < t_m and order n, the weights alpha solve
V^T alpha = mu with V_ki = t_k^(i-1) (k = 1..m, i = 1..n); for m > n the solution of
minimum 2-norm is selected.

Reading R1: the printed moment vector "(dt)^i/(i+1), i=1..n" is
index-shifted against the basis 1, t, ..., t^(n-1); we use mu_i = int_a^b tau^(i-1) dtau
= (b^i - a^i)/i, which reproduces the classical tableaux (pinned in
tests/test_oracle_abcoef.py against AB2/AB3/AB4 and the exact AB34 min-norm weights).

The minimum-norm solution is alpha = V (V^T V)^(-1) mu, computed here by exact Gaussian
elimination on Fractions; it is then rounded once to fp64 by the caller.
"""
from __future__ import annotations

from fractions import Fraction as Fr
from typing import Sequence


class DegenerateNodes(ValueError):
    pass


class InsufficientHistory(ValueError):
    pass


def _solve(A, rhs):
    """Exact Gauss-Jordan solve of the square system A x = rhs (lists of Fractions)."""
    n = len(A)
    M = [list(A[i]) + [rhs[i]] for i in range(n)]
    for col in range(n):
        piv = next((r for r in range(col, n) if M[r][col] != 0), None)
        if piv is None:
            raise DegenerateNodes("degenerate nodes")
        M[col], M[piv] = M[piv], M[col]
        p = M[col][col]
        M[col] = [v / p for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [vr - f * vc for vr, vc in zip(M[r], M[col])]
    return [M[i][n] for i in range(n)]


def ab_weights(nodes: Sequence, n: int, a, b):
    """Weights alpha_k (oldest node first) with sum_k alpha_k p(t_k) = int_a^b p for every
    polynomial p of degree < n; minimum 2-norm when m = len(nodes) > n."""
    t = [Fr(x) for x in nodes]
    m = len(t)
    if m < n:
        raise InsufficientHistory("insufficient history")
    if len(set(t)) != m:
        raise DegenerateNodes("degenerate nodes")
    a, b = Fr(a), Fr(b)
    V = [[tk ** i for i in range(n)] for tk in t]                  # m x n
    mu = [(b ** (i + 1) - a ** (i + 1)) / (i + 1) for i in range(n)]
    VtV = [[sum(V[k][i] * V[k][j] for k in range(m)) for j in range(n)] for i in range(n)]
    lam = _solve(VtV, mu)
    return [sum(V[k][i] * lam[i] for i in range(n)) for k in range(m)]


def uniform_nodes(m: int):
    """Nodes -(m-1), ..., -1, 0 (units of the mesh's own step), oldest first."""
    return [Fr(-(m - 1) + k) for k in range(m)]


def partial_weights(m: int, n: int, theta):
    """Weights integrating the degree-(n-1) extrapolant of the m uniform history values over
    [0, theta] (units of the mesh's step): the full AB step for theta = 1 and the
    'integrate the slow extrapolant partially' of MRAB Steps 2 and 5 otherwise."""
    return ab_weights(uniform_nodes(m), n, 0, theta)
