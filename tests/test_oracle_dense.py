"""Pin of the oracle's assembled RHS (oracle/rhs.py) against the dense brute-force reference
tests/dense_ref.py (explicit Kronecker-style D blocks per run, explicit SAT and interpolation
matrices, numerical eigendecomposition for K^+-), element by element, on small overset pairs
that contain far-field corners, hole edges, overset faces and their corners, a periodic
direction and an isothermal wall (SURVEY §8(c) pin "everything on tiny grids")."""
import math

import numpy as np
import pytest

import synth
from synth import configs as C
from oracle import overset, rhs as orhs
from dense_ref import DenseRHS


def _ogrid_pair():
    """Viscous O-grid 24 x 9 (r in [0.5, 2], wall at r = 0.5) over a 33^2 far-field box."""
    og = C._ogrid("ogrid", 24, 9, 0.5, 2.0, 1.05, 1, 1)
    bg = C._cart("background", (-4.0, -4.0), (4.0, 4.0), (33, 33), (False, False),
                 ((C.FARFIELD, C.FARFIELD), (C.FARFIELD, C.FARFIELD)), 0, 2)
    meshes = [og, bg]
    q0 = [C._uniform_state(m, 1.0, (0.2, 0.0), 1.0 / C.GAMMA) for m in meshes]
    return C.Problem("ogrid-pair", 2, meshes, q0, viscous=True, Re=50.0, Pr=0.72,
                     q_inf=C._qinf(2, 0.2), wall_T=1.0)


def _problems():
    return {"config1": synth.make_config(1), "config2-test": synth.make_config(2, "test"),
            "ogrid-pair": _ogrid_pair()}


@pytest.mark.parametrize("name", ["config1", "config2-test", "ogrid-pair"])
def test_oracle_rhs_equals_dense_reference(name):
    p = _problems()[name]
    st = orhs.build(p)
    dense = DenseRHS(p, st.ov)
    for g in range(len(p.meshes)):                     # receiver sets recomputed from the runs
        assert dense.receiver_points(g) == sorted(int(x) for x in st.ov.receivers[g].point)
    rng = np.random.default_rng(7)
    states = [q * (1.0 + 1e-2 * rng.standard_normal(q.shape)) for q in p.q0]
    Ro = orhs.rhs(p, st, states)
    Rd = dense.rhs(states)
    for g in range(len(p.meshes)):
        for c in range(4):
            scale = max(np.max(np.abs(Rd[g][c])), 1e-300)
            err = np.max(np.abs(Ro[g][c] - Rd[g][c])) / scale
            assert err <= 1e-12, (name, g, c, err)


def test_dense_reference_detects_a_dropped_sat_term():
    """Control: removing the wall SAT of one point changes the dense RHS there by O(1)."""
    p = _ogrid_pair()
    st = orhs.build(p)
    dense = DenseRHS(p, st.ov)
    rng = np.random.default_rng(8)
    states = [q * (1.0 + 1e-2 * rng.standard_normal(q.shape)) for q in p.q0]
    Ro = orhs.rhs(p, st, states)
    key = next(k for k, face in dense.ends[0][1].items() if face and k[1] > 0)   # a wall point
    del dense.ends[0][1][key]
    Rd = dense.rhs(states)
    pnt = key[0]
    diff = np.abs(Ro[0].reshape(4, -1)[:, pnt] - Rd[0].reshape(4, -1)[:, pnt]).max()
    assert diff > 1e-3 * np.abs(Ro[0]).max()
