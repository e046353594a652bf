"""Pin of the SAT readings R14-R16 (p0 = 17/48, K^+ on the kappa-min face, 1/p0 on every term,
far-field target q_inf) by the property they exist for: the linearised SBP-SAT semi-discretisation
about a uniform state is stable (SURVEY §8(c) pins: 'max Re lambda < 0' for 2-D single meshes,
Euler and viscous).  A wrong penalty sign or side makes the spectrum leave the left half plane,
which the SAT identities (tests/test_oracle_gas.py) alone would not catch.

The Jacobian dR/dq of the oracle's RHS is formed column by column by central differences on a
13 x 13 Cartesian mesh with far-field SAT on all four faces."""
import numpy as np
import pytest

import synth
from synth.configs import primitive_to_conserved
from oracle import rhs


def _tiny_problem(viscous, Re):
    p = synth.make_config(2, "test")
    m = p.meshes[0]
    n = 13
    x = np.linspace(-1.0, 1.0, n)
    X, Y = np.meshgrid(x, x)                 # [j][i]
    m.shape = (n, n)
    m.xyz = np.stack([X, Y])
    m.periodic = (False, False)
    m.face_bc = ((1, 1), (1, 1))
    p.meshes = [m]
    p.viscous = viscous
    p.Re = Re
    shp = (n, n)
    q = primitive_to_conserved(np.ones(shp), [np.full(shp, 0.5), np.full(shp, 0.2)], np.full(shp, 1 / 1.4))
    p.q0 = [q]
    p.q_inf = q.reshape(p.nc, -1)[:, 0].copy()
    return p


def _max_real_eig(p):
    st = rhs.build(p)
    q0 = p.q0[0]
    R0 = rhs.rhs(p, st, [q0])[0]
    assert np.max(np.abs(R0)) < 1e-11          # q = q_inf: every term vanishes
    nv = q0.size
    Jm = np.empty((nv, nv))
    eps = 1e-6
    flat = q0.reshape(-1)
    for k in range(nv):
        qp = flat.copy(); qp[k] += eps
        qm = flat.copy(); qm[k] -= eps
        Rp = rhs.rhs(p, st, [qp.reshape(q0.shape)])[0].reshape(-1)
        Rm = rhs.rhs(p, st, [qm.reshape(q0.shape)])[0].reshape(-1)
        Jm[:, k] = (Rp - Rm) / (2 * eps)
    lam = np.linalg.eigvals(Jm)
    return float(np.max(lam.real)), float(np.max(np.abs(lam)))


@pytest.mark.parametrize("viscous,Re", [(False, 1.0), (True, 100.0)])
def test_linearised_far_field_sat_is_stable(viscous, Re):
    mre, rad = _max_real_eig(_tiny_problem(viscous, Re))
    # stable: no eigenvalue in the right half plane beyond finite-difference noise
    assert mre < 1e-6 * rad, (mre, rad)


def test_flipped_penalty_side_is_unstable(monkeypatch):
    """Control: the same test detects a wrong reading.  Swapping the characteristic splitting
    (K^- on the kappa-min face instead of K^+) must push eigenvalues into the right half plane."""
    from oracle import gas
    orig = gas.k_matrix if hasattr(gas, "k_matrix") else None
    if orig is None:
        pytest.skip("oracle.gas.k_matrix not exposed")

    def flipped(q, n, side, *a, **kw):
        return orig(q, n, -side, *a, **kw)

    monkeypatch.setattr(gas, "k_matrix", flipped)
    mre, rad = _max_real_eig(_tiny_problem(False, 1.0))
    assert mre > 1e-3 * rad, (mre, rad)
