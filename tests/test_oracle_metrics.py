"""Pins of oracle/metrics.py (reading R3 of DESIGN.md)."""
import math

import numpy as np
import pytest

from oracle import metrics, sbp
import synth


def _positions(active, periodic):
    d = active.ndim
    return [sbp.segment_positions(active, d - 1 - k, periodic[k]) for k in range(d)]


def test_quadratic_map_2d_exact():
    """x = xi + 0.01 eta^2, y = eta + 0.02 xi^2 + 0.005 xi eta: D1 is exact for degree <= 2, so
    the metric terms equal the analytic cofactors."""
    n = 14
    xi, eta = np.meshgrid(np.arange(n, dtype=float), np.arange(n, dtype=float), indexing="xy")
    x = xi + 0.01 * eta ** 2
    y = eta + 0.02 * xi ** 2 + 0.005 * xi * eta
    xyz = np.stack([x, y])
    pos = _positions(np.ones((n, n), bool), (False, False))
    Jinv, M = metrics.metrics(xyz, ((0, 0), (0, 0)), pos)
    x_xi, x_eta = np.ones_like(x), 0.02 * eta
    y_xi, y_eta = 0.04 * xi + 0.005 * eta, 1.0 + 0.005 * xi
    assert np.allclose(Jinv, x_xi * y_eta - x_eta * y_xi, atol=1e-13)
    assert np.allclose(M[0][0], y_eta, atol=1e-13) and np.allclose(M[0][1], -x_eta, atol=1e-13)
    assert np.allclose(M[1][0], -y_xi, atol=1e-13) and np.allclose(M[1][1], x_xi, atol=1e-13)


def test_affine_map_3d():
    """Affine 3-D map x = A xi: J^-1 = det A and M = cofactor matrix (J^-1 A^-1 rows)."""
    n = 10
    A = np.array([[1.0, 0.2, 0.1], [0.05, 0.9, 0.3], [0.1, -0.2, 1.1]])
    g = np.meshgrid(*[np.arange(n, dtype=float)] * 3, indexing="ij")   # (k, j, i) numpy
    xi = np.stack([g[2], g[1], g[0]])
    xyz = np.einsum("ck,k...->c...", A, xi)
    pos = _positions(np.ones((n, n, n), bool), (False,) * 3)
    Jinv, M = metrics.metrics(xyz, ((0,) * 3,) * 3, pos)
    assert np.allclose(Jinv, np.linalg.det(A), atol=1e-12)
    cof = np.linalg.det(A) * np.linalg.inv(A)        # cof[kappa][i] = J^-1 dkappa/dx_i
    for k in range(3):
        for i in range(3):
            assert np.allclose(M[k][i], cof[k, i], atol=1e-12)


@pytest.mark.parametrize("cid,g", [(2, 1), (5, 0), (5, 1), (3, 0)])
def test_free_stream_preservation(cid, g):
    """sum_kappa D_kappa M[kappa][i] = 0 (the conservative forms preserve a uniform flow) on
    the hole-free curvilinear meshes of the workloads (incl. the periodic O-grid)."""
    p = synth.make_config(cid, "test")
    m = p.meshes[g]
    act = np.ones(tuple(reversed(m.shape)), bool)
    pos = _positions(act, m.periodic)
    Jinv, M = metrics.metrics(m.xyz, m.period, pos)
    assert Jinv.min() > 0
    for i in range(m.dim):
        div = sum(sbp.d1(M[k][i], metrics.axis_of(k, m.dim), *pos[k]) for k in range(m.dim))
        assert np.max(np.abs(div)) < 1e-12 * np.max(np.abs(M[0][0]))


def test_periodic_seam_cartesian():
    """Periodic Cartesian mesh: the seam unwrapping gives J^-1 = h_x h_y h_z everywhere."""
    p = synth.make_config(4, "test")
    m = p.meshes[0]
    act = np.ones(tuple(reversed(m.shape)), bool)
    Jinv, M = metrics.metrics(m.xyz, m.period, _positions(act, m.periodic))
    hx = m.xyz[0, 0, 0, 1] - m.xyz[0, 0, 0, 0]
    hy = m.xyz[1, 0, 1, 0] - m.xyz[1, 0, 0, 0]
    hz = m.xyz[2, 1, 0, 0] - m.xyz[2, 0, 0, 0]
    assert np.allclose(Jinv, hx * hy * hz, rtol=1e-13)
    assert np.allclose(M[0][0], hy * hz, rtol=1e-13) and np.allclose(M[0][1], 0, atol=1e-15)
