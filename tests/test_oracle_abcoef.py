"""Pins of oracle/abcoef.py and oracle/timeint.py.

AB tableaux and the min-norm extended-history weights, partial
integrals for MRAB, AB order of convergence on y' = lambda y, MRAB reductions
(SR = 1 == SRAB; decoupled == per-component SRAB), evaluation counts SR + 1 per
macro step, coupled-linear MRAB order ~ n (anchor: the printed EOCs
2.894-2.986 of P:986-1006).
"""
from fractions import Fraction as Fr
import math

import numpy as np
import pytest

from oracle import abcoef, timeint


def test_classical_tableaux():
    u = abcoef.uniform_nodes
    assert abcoef.ab_weights(u(2), 2, 0, 1) == [Fr(-1, 2), Fr(3, 2)]
    assert abcoef.ab_weights(u(3), 3, 0, 1) == [Fr(5, 12), Fr(-16, 12), Fr(23, 12)]
    assert abcoef.ab_weights(u(4), 4, 0, 1) == [Fr(-9, 24), Fr(37, 24), Fr(-59, 24), Fr(55, 24)]
    assert abcoef.ab_weights([0], 1, 0, 1) == [Fr(1)]                  # forward Euler


def test_min_norm_ab34():
    """AB34: moment conditions hold, alpha lies in range(V) (=> minimum norm), and the norm
    is below every zero-padded square solution."""
    t = abcoef.uniform_nodes(4)
    al = abcoef.ab_weights(t, 3, 0, 1)
    assert al == [Fr(43, 120), Fr(-79, 120), Fr(-31, 120), Fr(187, 120)]
    for i in range(3):
        assert sum(a * tk ** i for a, tk in zip(al, t)) == Fr(1, i + 1)
    nrm = sum(a * a for a in al)
    for drop in range(4):
        sub = [x for k, x in enumerate(t) if k != drop]
        sq = abcoef.ab_weights(sub, 3, 0, 1)
        assert nrm < sum(a * a for a in sq)


def test_errors():
    with pytest.raises(abcoef.InsufficientHistory):
        abcoef.ab_weights([0, 1], 3, 0, 1)
    with pytest.raises(abcoef.DegenerateNodes):
        abcoef.ab_weights([0, 0, 1], 3, 0, 1)


def test_partial_weights_additive_and_exact():
    """Partial integrals over [0, j/4] are additive and exact for degree < n."""
    for m, n in ((3, 3), (4, 3), (4, 4), (5, 4)):
        for j in range(1, 4):
            w = abcoef.partial_weights(m, n, Fr(j, 4))
            w_lo = abcoef.ab_weights(abcoef.uniform_nodes(m), n, 0, Fr(j - 1, 4))
            w_step = abcoef.ab_weights(abcoef.uniform_nodes(m), n, Fr(j - 1, 4), Fr(j, 4))
            assert [a + b for a, b in zip(w_lo, w_step)] == w
            for deg in range(n):
                lhs = sum(wk * tk ** deg for wk, tk in zip(w, abcoef.uniform_nodes(m)))
                assert lhs == Fr(j, 4) ** (deg + 1) / (deg + 1)
    # slow partial weights of AB3 over a quarter step (derived)
    assert abcoef.partial_weights(3, 3, Fr(1, 4)) == [Fr(7, 384), Fr(-13, 192), Fr(115, 384)]


class _Lin:
    """Linear ODE system y_g' = sum_h A[g][h] y_h for the time-integration pins."""

    def __init__(self, A, y0, n, m, h):
        self.A = np.asarray(A, dtype=np.float64)
        self.meshes = [type("M", (), {"step_multiple": 1})() for _ in range(len(y0))]
        self.q0 = [np.array([v], dtype=np.float64) for v in y0]
        self.order_n, self.history_m, self.h = n, m, h

    def rhs(self, states, which=None):
        y = np.array([s[0] for s in states])
        d = self.A @ y
        return [np.array([d[g]]) if (which is None or g in which) else None
                for g in range(len(states))]


def _run(sys_, steps, T):
    mr = timeint.MRAB(sys_, steps=steps, rhs_fn=sys_.rhs)
    S = max(steps)
    nmac = int(round(T / (S * sys_.h))) - (sys_.history_m - 1)
    mr.run(nmac)
    return mr, float(mr.t) * sys_.h


@pytest.mark.parametrize("n,m", [(2, 2), (3, 3), (3, 4), (4, 4), (4, 5)])
def test_ab_order_scalar(n, m):
    lam = -1.0
    errs = []
    hs = [0.05, 0.025, 0.0125]
    for h in hs:
        s = _Lin([[lam]], [1.0], n, m, h)
        mr, t = _run(s, [1], 2.5)
        errs.append(abs(mr.base[0][0] - math.exp(lam * t)))
    eoc = math.log(errs[1] / errs[2]) / math.log(2)
    assert abs(eoc - n) < 0.3, eoc


def _single_rate_vec(A, y0, h, nboot, nab):
    """Hand-written coupled single-rate AB3 (vector y' = A y): nboot Heun RK3 steps at h
    recording the stage-1 RHS of the last two of them, then AB3 at h."""
    A = np.asarray(A, dtype=np.float64)
    y = np.asarray(y0, dtype=np.float64)
    hist = []
    for k in range(nboot):
        k1 = A @ y
        k2 = A @ (y + h / 3 * k1)
        k3 = A @ (y + 2 * h / 3 * k2)
        if nboot - k <= 2:
            hist.append(k1)
        y = y + h * (k1 / 4 + 3 * k3 / 4)
    hist.append(A @ y)
    al = (5 / 12, -16 / 12, 23 / 12)
    for _ in range(nab):
        y = y + h * sum(a * f for a, f in zip(al, hist))
        hist = hist[1:] + [A @ y]
    return y


def test_sr1_equals_srab_and_counts():
    """MRAB with every step ratio 1 is single-rate AB: the oracle's MRAB on a coupled
    2-component system against an independent hand-written coupled AB3 driver."""
    A = [[-1.0, 0.1], [0.1, -0.05]]
    h, nmac = 0.01, 40
    s = _Lin(A, [1.0, 0.5], 3, 3, h)
    mr = timeint.MRAB(s, steps=[1, 1], rhs_fn=s.rhs)
    mr.run(nmac)
    ref = _single_rate_vec(A, [1.0, 0.5], h, 2, nmac)
    assert abs(mr.base[0][0] - ref[0]) <= 1e-14 and abs(mr.base[1][0] - ref[1]) <= 1e-14
    # counts: SR fast + 1 slow per macro step after the bootstrap
    for SR in (2, 3, 4):
        s = _Lin(A, [1.0, 0.5], 3, 3, 0.01)
        mr = timeint.MRAB(s, steps=[1, SR], rhs_fn=s.rhs)
        mr.bootstrap()
        c0 = list(mr.counts)
        for _ in range(5):
            mr.macro_step()
        assert mr.counts[0] - c0[0] == 5 * SR and mr.counts[1] - c0[1] == 5


def _heun(lam, y, h):
    k1 = lam * y
    k2 = lam * (y + h / 3 * k1)
    k3 = lam * (y + 2 * h / 3 * k2)
    return y + h * (k1 / 4 + 3 * k3 / 4), k1


def _single_rate_reference(lam, y0, h, every, nboot, nab):
    """Hand-written scalar driver: nboot Heun steps at h (recording the stage-1 RHS every
    `every` steps at the last two aligned times), then AB3 at step every*h."""
    y, hist = y0, []
    for k in range(nboot):
        left = nboot - k
        y_new, k1 = _heun(lam, y, h)
        if left % every == 0 and left // every <= 2:
            hist.append(k1)
        y = y_new
    hist.append(lam * y)
    al = (5 / 12, -16 / 12, 23 / 12)
    H = every * h
    for _ in range(nab):
        y = y + H * sum(a * f for a, f in zip(al, hist))
        hist = hist[1:] + [lam * y]
    return y


def test_decoupled_reduces_to_single_rate():
    """Decoupled components under MRAB equal each component integrated by single-rate AB3 at
    its own step after the same RK bootstrap (S:195 'decoupled system' reduction)."""
    h, SR, nmac = 0.01, 3, 10
    s = _Lin([[-1.0, 0.0], [0.0, -0.3]], [1.0, 2.0], 3, 3, h)
    mr = timeint.MRAB(s, steps=[1, SR], rhs_fn=s.rhs)
    mr.run(nmac)
    nboot = 2 * SR
    fast = _single_rate_reference(-1.0, 1.0, h, 1, nboot, nmac * SR)
    slow = _single_rate_reference(-0.3, 2.0, h, SR, nboot, nmac)
    assert abs(fast - mr.base[0][0]) <= 1e-14
    assert abs(slow - mr.base[1][0]) <= 1e-14


@pytest.mark.parametrize("steps,n,m", [((1, 2), 3, 3), ((1, 4), 3, 3), ((1, 4), 3, 4),
                                        ((1, 2, 4, 8), 4, 4), ((1, 2, 4, 8), 2, 2)])
def test_coupled_mrab_order(steps, n, m):
    """Coupled linear system f' = -f + 0.1 s, s' = -0.05 s + 0.1 f, EOC ~ n."""
    G = len(steps)
    A = np.full((G, G), 0.1)
    for g in range(G):
        A[g, g] = -1.0 / (1 + 3 * g)
    y0 = [1.0 - 0.2 * g for g in range(G)]
    from scipy.linalg import expm
    errs = []
    Hs = [0.04, 0.02, 0.01]
    for H in Hs:
        s = _Lin(A, y0, n, m, H / max(steps))
        mr, t = _run(s, list(steps), 2.0)
        ex = expm(A * t) @ np.array(y0)
        errs.append(max(abs(mr.base[g][0] - ex[g]) for g in range(G)))
    eoc = math.log(errs[1] / errs[2]) / math.log(2)
    assert abs(eoc - n) < 0.3, (eoc, errs)
