"""Step-matrix stability procedure (ORACLE, test infrastructure).

PAPER.md §5.1 "Procedure for Determining Discrete Stability":
  phi_{n+1} ~ G_eps phi_n                                              (eq:sm)
  G_eps(:, j) ~ (phi_{n+1,mod} - phi_{n+1,base}) / eps,  phi_mod = phi + eps e_j   (eq:sm_form)
  "the stability vector element being perturbed may also be a right-hand side history
  element"; eps = 1e-7; stable iff rho(G_eps) <= 1 (SLEPc Krylov-Schur there, a dense
  eigensolve here: the oracle forms every column).
§5.2-5.4: the maximum stable timestep is found by bisection to 1e-4.

Integrator vector (reading R-SM): at a macro boundary t the vector of mesh g is
its state y_g and its m-1 RHS history entries R_g(t - (m-1-k) h_g), k = 0..m-2 (oldest first).
R_g(t) itself is a function of the states (it is re-evaluated from them), so it is not a free
element.  One application of the map = one MRAB macro step (timeint.MRAB, fastest-first, no
re-extrapolation), after which the vector is (y_g(t+H), R_g(t+H-(m-1-k) h_g)).
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np

from . import timeint

EPS = 1e-7


def pack(states, hists):
    """states[g]: array; hists[g]: list of m-1 arrays (oldest first) -> flat phi."""
    parts = []
    for y, H in zip(states, hists):
        parts.append(np.asarray(y, dtype=np.float64).ravel())
        parts.extend(np.asarray(r, dtype=np.float64).ravel() for r in H)
    return np.concatenate(parts)


def unpack(phi, shapes, m):
    """Inverse of pack for per-mesh array shapes."""
    states, hists, o = [], [], 0
    for shp in shapes:
        n = int(np.prod(shp))
        states.append(phi[o:o + n].reshape(shp).copy())
        o += n
        H = []
        for _ in range(m - 1):
            H.append(phi[o:o + n].reshape(shp).copy())
            o += n
        hists.append(H)
    assert o == phi.size
    return states, hists


def macro_map(problem, phi, steps=None, setup=None, rhs_fn=None):
    """One MRAB macro step applied to the integrator vector phi (see module docstring)."""
    mr = timeint.MRAB(problem, setup=setup, steps=steps, rhs_fn=rhs_fn)
    shapes = [np.shape(q) for q in problem.q0]
    ys, Hs = unpack(phi, shapes, mr.m)
    R = mr.rhs_fn(ys)                       # R_g(t) from the states (Step 1's newest entries)
    G = len(ys)
    mr.base = [y.copy() for y in ys]
    mr.rings = [list(Hs[g]) + [R[g]] for g in range(G)]
    mr.t = Fr(0)
    mr.tg = [Fr(0)] * G
    mr.macro_step()
    return pack(mr.base, [mr.rings[g][:-1] for g in range(G)])


def step_matrix(problem, phi0, eps=EPS, steps=None, setup=None, rhs_fn=None):
    """G_eps column by column (eq:sm_form)."""
    base = macro_map(problem, phi0, steps, setup, rhs_fn)
    G = np.empty((base.size, phi0.size))
    for j in range(phi0.size):
        ph = phi0.copy()
        ph[j] += eps
        G[:, j] = (macro_map(problem, ph, steps, setup, rhs_fn) - base) / eps
    return G


def spectral_radius(G):
    """rho(G) = max |lambda| (dense eigensolve)."""
    return float(np.max(np.abs(np.linalg.eigvals(G))))


def max_stable(rho_of, lo, hi, tol=1e-4):
    """Largest x in [lo, hi] with rho_of(x) <= 1, by bisection to `tol`;
    rho_of(lo) must be <= 1."""
    assert rho_of(lo) <= 1.0
    if rho_of(hi) <= 1.0:
        return hi
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if rho_of(mid) <= 1.0:
            lo = mid
        else:
            hi = mid
    return lo
