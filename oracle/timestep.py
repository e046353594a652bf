"""Stable-timestep estimate (ORACLE, test infrastructure).

PAPER.md §4.1 eq:ts_inv / eq:ts_visc / eq:ts_overall: per mesh point

  dt_inv  = J^-1 / ( sum_i |U . (1/J) d xi_i/dx| + c sqrt(xi_hat . xi_hat) )
  dt_visc = J^-1 / ( [the same] + 2 nu* J ( sum_i sqrt((1/J) d xi_i/dx . (1/J) d xi_i/dx) )^2 )
  dt      = min(dt_inv, dt_visc), then the minimum over all mesh points.

The printed eq:ts_visc has an unbalanced parenthesis and xi_hat is not defined; reading R20
(SURVEY G20): with M_i = J^-1 grad(xi_i) (the metric rows of oracle.metrics)

  dt = J^-1 / [ sum_i ( |U . M_i| + c |M_i| ) + 2 nu* J ( sum_i |M_i| )^2 ],
  nu* = max(mu, k/c_v) / rho = max(1, gamma/Pr) / (rho Re)   (mu = 1, R11),

the last term only for viscous problems (for Euler dt = dt_inv).  Since the viscous term is
non-negative, min(dt_inv, dt_visc) = dt_visc wherever it applies; both are formed and the
minimum taken, as the paper states.

Pins (tests/test_oracle_timestep.py): the textbook Cartesian CFL formula
1 / ((|u|+c)/dx + (|v|+c)/dy) typed in the test; the viscous Cartesian closed form; the
finest micro steps h = 0.5 min dt of the five synthetic configs printed in SURVEY.md §8(d).
"""
from __future__ import annotations

import numpy as np

from . import gas


def dt_field(problem, setup, g, q):
    """dt at every point of mesh g for the state q (nc, *spatial); inactive points get +inf."""
    d = problem.dim
    geo = setup.geom[g]
    rho, u, p, T = gas.primitives(q, problem.gamma)
    c = np.sqrt(problem.gamma * p / rho)
    conv = np.zeros_like(rho)
    msum = np.zeros_like(rho)
    for i in range(d):
        Un = sum(u[k] * geo.M[i][k] for k in range(d))
        Mn = np.sqrt(sum(geo.M[i][k] * geo.M[i][k] for k in range(d)))
        conv = conv + np.abs(Un) + c * Mn
        msum = msum + Mn
    with np.errstate(divide="ignore", invalid="ignore"):
        dt_inv = geo.Jinv / conv
        dt = dt_inv
        if problem.viscous:
            nu = max(1.0, problem.gamma / problem.Pr) / (rho * problem.Re)
            dt_visc = geo.Jinv / (conv + 2.0 * nu * geo.J * msum * msum)
            dt = np.minimum(dt_inv, dt_visc)
    return np.where(geo.active, dt, np.inf)


def dt_min(problem, setup, states):
    """Per-mesh minimum of dt over the active points (eq:ts_overall and the final min)."""
    return [float(np.min(dt_field(problem, setup, g, q))) for g, q in enumerate(states)]


def macro_step(problem, setup, states, cfl):
    """Largest macro step H with s_g H / S <= cfl dt_g on every mesh (h = H / SR)."""
    S = max(m.step_multiple for m in problem.meshes)
    dts = dt_min(problem, setup, states)
    return cfl * S * min(dt / m.step_multiple for dt, m in zip(dts, problem.meshes))
