"""Pins of the slowest-first MRAB variants oracle.timeint.MRAB.macro_step_sf (P:536-548,
reading R-SF): closed forms of one first-order macro step typed here (they separate the three
schemes and fix which state each evaluation sees), reductions (decoupled system and SR = 1
against hand-written single-rate AB3 drivers), evaluation counts, order of convergence."""
import math

import numpy as np
import pytest

from oracle import timeint
from test_oracle_abcoef import _Lin, _single_rate_reference, _single_rate_vec


def _euler_mr(A, f0, s0, h, scheme):
    """One macro step (SR = 2, n = m = 1) by hand; returns f2, s2 and the new history values."""
    (a, b), (c, d) = A
    Rf0, Rs0 = a * f0 + b * s0, c * f0 + d * s0
    s2 = s0 + 2 * h * Rs0
    f1 = f0 + h * Rf0
    if scheme == "fastest_first":
        s1 = s0 + h * Rs0
        f2 = f1 + h * (a * f1 + b * s1)
        return f2, s2, a * f2 + b * s2, c * f2 + d * s2
    ft2 = f0 + 2 * h * Rf0                       # fast extrapolated over the macro step
    Rs2 = c * ft2 + d * s2                       # slow evaluated first
    s1 = s0 + h * (Rs2 if scheme == "slowest_first_reextrap" else Rs0)
    f2 = f1 + h * (a * f1 + b * s1)
    return f2, s2, a * f2 + b * s2, Rs2


@pytest.mark.parametrize("scheme", ["fastest_first", "slowest_first", "slowest_first_reextrap"])
def test_first_order_closed_form(scheme):
    A = [[-1.0, 0.4], [0.3, -0.2]]
    h = 0.05
    s = _Lin(A, [1.0, 0.5], 1, 1, h)
    mr = timeint.MRAB(s, steps=[1, 2], rhs_fn=s.rhs)
    mr.bootstrap()                               # m - 1 = 0 RK steps: histories = RHS at q0
    mr.run(1, scheme=scheme)
    f2, s2, Rf2, Rs2 = _euler_mr(A, 1.0, 0.5, h, scheme)
    assert abs(mr.base[0][0] - f2) <= 1e-15 and abs(mr.base[1][0] - s2) <= 1e-15
    assert abs(mr.rings[0][-1][0] - Rf2) <= 1e-15 and abs(mr.rings[1][-1][0] - Rs2) <= 1e-15
    # the three schemes differ on this system
    others = [x for x in ("fastest_first", "slowest_first", "slowest_first_reextrap") if x != scheme]
    for o in others:
        assert abs(_euler_mr(A, 1.0, 0.5, h, o)[0] - f2) > 1e-6 or abs(_euler_mr(A, 1.0, 0.5, h, o)[3] - Rs2) > 1e-6


@pytest.mark.parametrize("reextrap", [False, True])
def test_decoupled_reduces_to_single_rate(reextrap):
    h, SR, nmac = 0.01, 3, 10
    s = _Lin([[-1.0, 0.0], [0.0, -0.3]], [1.0, 2.0], 3, 3, h)
    mr = timeint.MRAB(s, steps=[1, SR], rhs_fn=s.rhs)
    mr.bootstrap()
    for _ in range(nmac):
        mr.macro_step_sf(reextrap)
    fast = _single_rate_reference(-1.0, 1.0, h, 1, 2 * SR, nmac * SR)
    slow = _single_rate_reference(-0.3, 2.0, h, SR, 2 * SR, nmac)
    assert abs(fast - mr.base[0][0]) <= 1e-14 and abs(slow - mr.base[1][0]) <= 1e-14
    # SR + 1 evaluations per macro step, as fastest-first
    assert mr.counts[0] - (2 * SR * 3 + 1) == nmac * SR and mr.counts[1] - (2 * SR * 3 + 1) == nmac


@pytest.mark.parametrize("reextrap", [False, True])
@pytest.mark.parametrize("order", [(1, 2), (2, 1)])
def test_order_of_convergence(reextrap, order):
    from scipy.linalg import expm
    A = np.array([[-1.0, 0.1], [0.1, -0.05]])
    if order == (2, 1):
        A = A[::-1, ::-1].copy()
    y0 = [1.0, 0.5]
    errs = []
    for H in (0.04, 0.02, 0.01):
        SR = 2
        s = _Lin(A, y0, 3, 3, H / SR)
        mr = timeint.MRAB(s, steps=[SR if o == 2 else 1 for o in order], rhs_fn=s.rhs)
        mr.bootstrap()
        while float(mr.t) * s.h < 2.0 - 1e-12:
            mr.macro_step_sf(reextrap)
        ex = expm(A * float(mr.t) * s.h) @ np.array(y0)
        errs.append(max(abs(mr.base[g][0] - ex[g]) for g in range(2)))
    eoc = math.log(errs[1] / errs[2]) / math.log(2)
    assert abs(eoc - 3) < 0.3, (eoc, errs)


def test_rejects_more_than_two_rates():
    s = _Lin(np.eye(3) * -1.0, [1.0, 1.0, 1.0], 3, 3, 0.01)
    mr = timeint.MRAB(s, steps=[1, 2, 4], rhs_fn=s.rhs)
    mr.bootstrap()
    with pytest.raises(ValueError):
        mr.macro_step_sf()
