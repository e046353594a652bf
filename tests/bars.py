"""Parity bars shared by the GPU tests (test infrastructure; may call oracle/).

Two kinds of bar, both per component ("Also report the per-component
version"):

* states (north_star: 1e-10 relative max-norm).  A single global denominator lets a small
  component (config 3's rho v ~ 1e-4 against max |rho E| ~ 1.8) be wrong at 1e-6 of its own
  size.  Each component c is therefore held to 1e-10 of its own natural scale:
      |Q_gpu - Q_orc|_c <= 1e-10 * scale_c,
      scale_rho = max|rho|, scale_rhoE = max|rho E|, scale_{rho u_i} = max|rho| * max c,
  i.e. momentum is measured in units of rho * (speed of sound), the acoustic scaling the
  nondimensionalisation fixes (c_inf = 1, reading R12).  A component at rest (rho v = 0 at
  t0 in config 4) would otherwise have a denominator of pure rounding noise.

* right-hand sides.  R = -J sum_kappa D_kappa Fhat_kappa cancels terms of size
  J |D| |Fhat| down to |R| (near-uniform states: |F|/h against |R| ~ 1e-4 |F|/h), so the
  rounding error of ANY correct evaluation order is eps * (sum of |terms|), not eps * |R|.
  The bar keeps 1e-12 but normalises each component by that cancellation scale:
      |R_gpu - R_orc|_c <= 1e-12 * max(max|R_orc,c|, S_c),
      S_c = max J * Dabs * sum_kappa max |Fhat_kappa,c|,
  Dabs = the largest absolute row sum of the 2-4 D1 (closure row 0: 24/17 + 59/34 + 4/17 +
  3/34 = 3.47).  1e-12 leaves ~1e4 ulps of headroom over eps * S_c.
"""
from __future__ import annotations

import numpy as np

from oracle import gas, rhs as orhs, sbp

STATE_BAR = 1e-10
RHS_BAR = 1e-12


def rel_global(a_list, b_list):
    """The north_star's relative max-norm (one denominator over meshes and components)."""
    num = max(float(np.max(np.abs(a - b))) for a, b in zip(a_list, b_list))
    den = max(float(np.max(np.abs(b))) for b in b_list)
    return num / den


def _dabs():
    D = sbp.d1_matrix(24)
    return float(max(sum(abs(float(x)) for x in row) for row in D))


def state_scales(q_list, gamma):
    nc = q_list[0].shape[0]
    d = nc - 2
    rho = max(float(np.max(np.abs(q[0]))) for q in q_list)
    cmax = 0.0
    for q in q_list:
        r, u, p, T = gas.primitives(q.reshape(nc, -1), gamma)
        cmax = max(cmax, float(np.sqrt(np.max(np.abs(T)))))
    sc = [rho] + [rho * cmax] * d + [max(float(np.max(np.abs(q[d + 1]))) for q in q_list)]
    return np.array(sc)


def state_errors(gpu, orc, gamma):
    """Per-component error / scale (each must be <= STATE_BAR)."""
    nc = orc[0].shape[0]
    sc = state_scales(orc, gamma)
    err = np.array([max(float(np.max(np.abs(a[c] - b[c]))) for a, b in zip(gpu, orc))
                    for c in range(nc)])
    return err / sc


def assert_states(gpu, orc, gamma, bar=STATE_BAR):
    g = rel_global(gpu, orc)
    pc = state_errors(gpu, orc, gamma)
    assert g <= bar and np.all(pc <= bar), (g, pc.tolist())
    return g, pc


def rhs_scales(p, st, states):
    """S_c of the module docstring, maximised over the meshes."""
    nc = p.nc
    dabs = _dabs()
    S = np.zeros(nc)
    for g, q in enumerate(states):
        geo = st.geom[g]
        FV = orhs.cartesian_viscous_fluxes(p, st, g, q)
        Fh = orhs.contravariant_fluxes(p, geo, q, FV)
        act = geo.active
        Jm = float(np.max(np.abs(geo.J[act])))
        for c in range(nc):
            s = sum(float(np.max(np.abs(F[c][act]))) for F in Fh)
            S[c] = max(S[c], Jm * dabs * s)
    return S


def rhs_errors(p, st, states, Rg, Ro):
    nc = p.nc
    S = rhs_scales(p, st, states)
    out = np.zeros(nc)
    for c in range(nc):
        err = max(float(np.max(np.abs(a[c] - b[c]))) for a, b in zip(Rg, Ro))
        den = max(max(float(np.max(np.abs(b[c]))) for b in Ro), S[c])
        out[c] = err / den
    return out


def assert_rhs(p, st, states, Rg, Ro, bar=RHS_BAR, global_bar=1e-10):
    g = rel_global(Rg, Ro)
    pc = rhs_errors(p, st, states, Rg, Ro)
    assert g <= global_bar and np.all(pc <= bar), (g, pc.tolist())
    return g, pc
