"""Pins of oracle/sbp.py against what the paper and the mathematics fix (not against itself).

P:205-208 / P:797-802 / P:1526-1544: diagonal-norm SBP operator, periodic symbol maximum
1.3722, RK4 limit on 61-point advection, global orders p+1/2 and p-1/2 in the discrete L2
norm of eq:l2error.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import sbp


@pytest.mark.parametrize("n", [8, 9, 12, 21])
def test_sbp_property_exact(n):
    """H D + D^T H = B = diag(-1, 0, ..., 0, 1) exactly in rationals (SBP definition)."""
    D = sbp.d1_matrix(n)
    H = sbp.h_matrix(n)
    for r in range(n):
        for c in range(n):
            q = H[r] * D[r][c] + D[c][r] * H[c]
            expect = Fr(-1) if r == c == 0 else Fr(1) if r == c == n - 1 else Fr(0)
            assert q == expect, (r, c, q)


def test_polynomial_exactness():
    """Boundary rows exact to degree 2, interior rows to degree 4 (2-4 operator)."""
    n = 16
    D = sbp.d1_matrix(n)
    for deg in range(0, 5):
        f = [Fr(i) ** deg for i in range(n)]
        df = [deg * Fr(i) ** (deg - 1) if deg else Fr(0) for i in range(n)]
        for r in range(n):
            val = sum(D[r][c] * f[c] for c in range(n))
            boundary = r < 4 or r > n - 5
            if deg <= 2 or not boundary:
                assert val == df[r], (deg, r)
    # and NOT exact for degree 3 on the boundary rows (it is a 2nd-order closure)
    f = [Fr(i) ** 3 for i in range(n)]
    assert sum(D[0][c] * f[c] for c in range(n)) != 0


def test_periodic_symbol_max():
    """max eigenvalue of the periodic operator lambda_max dx = 1.3722 i."""
    n = 61
    D = np.array([[float(v) for v in row] for row in sbp.d1_matrix(n, periodic=True)])
    lam = np.linalg.eigvals(D)
    assert np.max(np.abs(lam.real)) < 1e-12
    # the 61 discrete modes sample the symbol; its maximum 1.3722 bounds them from above
    assert 1.3722 - 2e-3 < np.max(np.abs(lam.imag)) <= 1.37223
    # continuous symbol: (4/3) sin t - (1/6) sin 2t, max at cos t = (2 - sqrt 6)/2
    t = np.arccos((2 - np.sqrt(6)) / 2)
    assert abs((4 / 3) * np.sin(t) - (1 / 6) * np.sin(2 * t) - 1.37222) < 1e-4


def test_rk4_advection_limit():
    """1-D periodic advection, 61 points on [0, 1.01666]: RK4 max stable dt is
    between 0.03 and 0.035 (found here by bisection on the RK4 amplification polynomial)."""
    n = 61
    dx = 1.01666 / n
    D = np.array([[float(v) for v in row] for row in sbp.d1_matrix(n, periodic=True)]) / dx
    lam = np.linalg.eigvals(-D)

    def stable(dt):
        z = lam * dt
        g = 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
        return np.all(np.abs(g) <= 1 + 1e-12)

    lo, hi = 0.01, 0.1
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if stable(mid) else (lo, mid)
    assert 0.03 < lo < 0.035


def _brute_positions(act, periodic):
    n = len(act)
    a = np.full(n, -1)
    b = np.full(n, -1)
    for i in range(n):
        if not act[i]:
            continue
        if periodic and act.all():
            a[i] = b[i] = sbp.FAR
            continue
        k, j = 0, i
        while True:
            jp = j - 1
            if jp < 0:
                if not periodic:
                    break
                jp += n
            if not act[jp]:
                break
            k += 1
            j = jp
        a[i] = k
        k, j = 0, i
        while True:
            jn = j + 1
            if jn >= n:
                if not periodic:
                    break
                jn -= n
            if not act[jn]:
                break
            k += 1
            j = jn
        b[i] = k
    return a, b


@pytest.mark.parametrize("periodic", [False, True])
def test_segment_positions_bruteforce(periodic):
    rng = np.random.default_rng(0)
    for _ in range(30):
        n = int(rng.integers(10, 40))
        act = rng.random(n) > 0.15
        if rng.random() < 0.2:
            act[:] = True
        a, b = sbp.segment_positions(act[None, :], 1, periodic)
        ea, eb = _brute_positions(act, periodic)
        assert np.array_equal(a[0], ea) and np.array_equal(b[0], eb)


@pytest.mark.parametrize("periodic", [False, True])
def test_d1_matches_dense_segments(periodic):
    """The vectorised segmented D1 equals the dense per-segment matrices (brute force)."""
    rng = np.random.default_rng(1)
    n = 40
    act = np.ones(n, dtype=bool)
    act[14:17] = False
    if periodic:
        act[33:35] = False            # a segment wraps the seam
    f = rng.standard_normal(n)
    a, b = sbp.segment_positions(act[None], 1, periodic)
    got = sbp.d1(f[None], 1, a, b)[0]
    expect = np.zeros(n)
    idx = np.nonzero(act)[0]
    # split active indices into cyclic runs
    runs, cur = [], [idx[0]]
    for i in idx[1:]:
        if i == cur[-1] + 1:
            cur.append(i)
        else:
            runs.append(cur)
            cur = [i]
    runs.append(cur)
    if periodic and runs[0][0] == 0 and runs[-1][-1] == n - 1 and len(runs) > 1:
        runs[0] = runs[-1] + runs[0]
        runs.pop()
    for run in runs:
        Dm = np.array([[float(v) for v in row] for row in sbp.d1_matrix(len(run))])
        expect[run] = Dm @ f[run]
    assert np.allclose(got, expect, rtol=0, atol=1e-14)


def test_global_order_discrete_l2():
    """in eq:l2error the global order is p + 1/2 for D1 and p - 1/2 for D1 D1
    (p = 2 boundary order); measured here on sin on non-periodic grids."""
    errs1, errs2, hs = [], [], []
    for n in (41, 81, 161, 321):
        x = np.linspace(0, 1, n)
        h = x[1] - x[0]
        f = np.sin(2 * np.pi * x + 0.3)
        act = np.ones((1, n), dtype=bool)
        a, b = sbp.segment_positions(act, 1, False)
        d1 = sbp.d1(f[None], 1, a, b)[0] / h
        d2 = sbp.d1(d1[None], 1, a, b)[0] / h
        e1 = d1 - 2 * np.pi * np.cos(2 * np.pi * x + 0.3)
        e2 = d2 + (2 * np.pi) ** 2 * np.sin(2 * np.pi * x + 0.3)
        errs1.append(np.sqrt(np.sum(e1 ** 2) * h))
        errs2.append(np.sqrt(np.sum(e2 ** 2) * h))
        hs.append(h)
    eoc1 = np.log(errs1[-2] / errs1[-1]) / np.log(hs[-2] / hs[-1])
    eoc2 = np.log(errs2[-2] / errs2[-1]) / np.log(hs[-2] / hs[-1])
    assert abs(eoc1 - 2.5) < 0.1
    assert abs(eoc2 - 1.5) < 0.1
