"""Pins of oracle/timestep.py (eq:ts, reading R20) and of the variable-macro-step
MRAB oracle.timeint.MRAB.macro_step_var.

timestep: the textbook Cartesian CFL formula and the viscous Cartesian closed form typed here;
the finest micro steps h = 0.5 min dt printed in SURVEY.md §8(d) for configs 1 and 2 (8.91e-3,
1.50e-3; computed there by the surveyor's scratch script, not by this oracle).
variable step: (a) constant H reproduces the fixed-step scheme; (b) a right-hand side that is
a polynomial of degree < n in time is integrated exactly whatever the step sequence (catches a
misplaced or dropped history node); (c) hand-written variable-step AB2 driver typed here;
(d) order n on a coupled linear system under a smoothly varying step."""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import synth
from oracle import rhs as orhs, timeint, timestep


def _uniform(p, rho, vel, pr):
    return [synth.configs.primitive_to_conserved(np.full(m.shape[::-1], rho), [np.full(m.shape[::-1], v) for v in vel],
                                                 np.full(m.shape[::-1], pr), p.gamma) for m in p.meshes]


def test_cartesian_cfl_closed_form():
    p = synth.make_config(1, "test")          # two Cartesian meshes, Euler
    st = orhs.build(p)
    rho, u, v, pr = 1.3, 0.4, -0.25, 0.9
    q = _uniform(p, rho, (u, v), pr)
    c = math.sqrt(p.gamma * pr / rho)
    for g, m in enumerate(p.meshes):
        x, y = m.xyz
        dx, dy = x[0, 1] - x[0, 0], y[1, 0] - y[0, 0]
        want = 1.0 / ((abs(u) + c) / dx + (abs(v) + c) / dy)
        got = timestep.dt_field(p, st, g, q[g])
        act = st.geom[g].active
        assert np.allclose(got[act], want, rtol=1e-12)
        assert np.all(np.isinf(got[~act]))


def test_cartesian_viscous_closed_form():
    p = synth.make_config(4, "test")          # 3-D Cartesian, viscous (Re 500)
    st = orhs.build(p)
    rho, vel, pr = 0.8, (0.3, 0.1, -0.2), 0.75
    q = _uniform(p, rho, vel, pr)
    c = math.sqrt(p.gamma * pr / rho)
    nu = max(1.0, p.gamma / p.Pr) / (rho * p.Re)
    for g, m in enumerate(p.meshes):
        X = m.xyz
        d = [X[0][0, 0, 1] - X[0][0, 0, 0], X[1][0, 1, 0] - X[1][0, 0, 0], X[2][1, 0, 0] - X[2][0, 0, 0]]
        conv = sum((abs(vel[i]) + c) / d[i] for i in range(3))
        want = 1.0 / (conv + 2.0 * nu * sum(1.0 / x for x in d) ** 2)
        got = timestep.dt_field(p, st, g, q[g])
        act = st.geom[g].active
        assert np.allclose(got[act], want, rtol=1e-10)


@pytest.mark.parametrize("cid,h", [(1, 8.91e-3), (2, 1.50e-3)])
def test_survey_micro_steps(cid, h):
    """SURVEY.md §8(d) 'Expected finest micro step' (CFL 0.5 on the finest mesh, ICs of §8(d))."""
    p = synth.make_config(cid, "full")
    st = orhs.build(p)
    got = 0.5 * min(timestep.dt_min(p, st, p.q0))
    assert abs(got - h) <= 0.006 * h, got


class _Sys:
    def __init__(self, rhs, y0, n, m, h):
        self.rhs = rhs
        self.meshes = [type("M", (), {"step_multiple": 1})() for _ in y0]
        self.q0 = [np.array([v], dtype=np.float64) for v in y0]
        self.order_n, self.history_m, self.h = n, m, h


def _lin(A):
    A = np.asarray(A, dtype=np.float64)

    def rhs(states, which=None):
        d = A @ np.array([s[0] for s in states])
        return [np.array([d[g]]) if (which is None or g in which) else None for g in range(len(states))]
    return rhs


def test_constant_H_reproduces_fixed_step():
    A = [[-1.0, 0.1], [0.1, -0.05]]
    for steps, n, m in (((1, 4), 3, 3), ((1, 2), 3, 4), ((1, 2, 4, 8), 4, 4)):
        G = len(steps)
        Ag = np.full((G, G), 0.1) - np.diag([1.0 / (1 + g) for g in range(G)])
        y0 = [1.0 - 0.1 * g for g in range(G)]
        h = 0.01
        a = timeint.MRAB(_Sys(_lin(Ag), y0, n, m, h), steps=list(steps), rhs_fn=_lin(Ag))
        b = timeint.MRAB(_Sys(_lin(Ag), y0, n, m, h), steps=list(steps), rhs_fn=_lin(Ag))
        a.run(6)
        b.bootstrap()
        for _ in range(6):
            b.macro_step_var(max(steps) * h)
        for g in range(G):
            assert abs(a.base[g][0] - b.base[g][0]) <= 1e-14


@pytest.mark.parametrize("steps,n,m", [((1, 2), 3, 3), ((1, 3), 3, 4), ((2, 1), 2, 2), ((1, 2, 4), 4, 4)])
def test_polynomial_forcing_is_exact(steps, n, m):
    """Mesh 0 carries a' = 1 (a = t); every other mesh g carries b_g' = (g+1) a^(n-1): its RHS
    is a polynomial of degree n-1 in time, which AB of order n integrates exactly from exact
    history, for any sequence of macro steps, at every rate (the coupling value a(t_j) comes
    from the partial integral of a constant, exact)."""
    G = len(steps)

    def rhs(states, which=None):
        a = states[0][0]
        out = [np.array([1.0])] + [np.array([(g + 1) * a ** (n - 1)]) for g in range(1, G)]
        return [out[g] if (which is None or g in which) else None for g in range(G)]

    S, h = max(steps), 0.01
    mr = timeint.MRAB(_Sys(rhs, [0.0] * G, n, m, h), steps=list(steps), rhs_fn=rhs)
    # exact start-up: states and histories on the exact solution (no RK error)
    t0 = (m - 1) * S * h
    mr.t = Fr((m - 1) * S)
    mr.tg = [mr.t] * G
    mr.base = [np.array([t0])] + [np.array([(g + 1) * t0 ** n / n]) for g in range(1, G)]
    for g in range(G):
        ts = [t0 - (m - 1 - k) * steps[g] * h for k in range(m)]
        mr.rings[g] = [np.array([1.0]) if g == 0 else np.array([(g + 1) * t ** (n - 1)]) for t in ts]
    t = t0
    for i, f in enumerate((1.0, 1.3, 0.7, 1.1, 0.55, 1.45, 0.9)):
        H = S * h * f
        mr.macro_step_var(H)
        t += H
        assert abs(mr.base[0][0] - t) <= 1e-13
        for g in range(1, G):
            assert abs(mr.base[g][0] - (g + 1) * t ** n / n) <= 2e-13 * max(1.0, t ** n), (i, g)


def test_variable_ab2_hand_driver():
    """Single-rate variable-step AB2, y_{k+1} = y_k + h_k [(1 + r/2) f_k - (r/2) f_{k-1}],
    r = h_k / h_{k-1} (textbook), against macro_step_var with S = 1."""
    lam, h = -0.7, 0.02
    s = _Sys(_lin([[lam]]), [1.0], 2, 2, h)
    mr = timeint.MRAB(s, steps=[1], rhs_fn=s.rhs)
    mr.bootstrap()
    y, f_old, f_new, h_old = mr.base[0][0], mr.rings[0][0][0], mr.rings[0][1][0], h
    for f in (1.2, 0.8, 1.5, 0.6, 1.0):
        hk = h * f
        r = hk / h_old
        y = y + hk * ((1 + r / 2) * f_new - (r / 2) * f_old)
        f_old, f_new, h_old = f_new, lam * y, hk
        mr.macro_step_var(hk)
        assert abs(mr.base[0][0] - y) <= 1e-15


def test_variable_step_order():
    A = np.array([[-1.0, 0.1], [0.1, -0.05]])
    from scipy.linalg import expm
    errs = []
    for H0 in (0.04, 0.02, 0.01):
        s = _Sys(_lin(A), [1.0, 0.5], 3, 3, H0 / 4)
        mr = timeint.MRAB(s, steps=[1, 4], rhs_fn=s.rhs)
        mr.bootstrap()
        t = float(mr.t) * s.h
        while t < 2.0:
            H = H0 * (1.0 + 0.3 * math.sin(3.0 * t))
            mr.macro_step_var(H)
            t += H
        ex = expm(A * float(mr.time)) @ np.array([1.0, 0.5])
        errs.append(max(abs(mr.base[g][0] - ex[g]) for g in range(2)))
    eoc = math.log(errs[1] / errs[2]) / math.log(2)
    assert abs(eoc - 3) < 0.35, (eoc, errs)
