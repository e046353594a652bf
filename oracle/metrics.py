"""Curvilinear metric terms (ORACLE, test infrastructure).

PAPER.md §4.1 uses the metric terms (1/J) d xi_i / d x of
[maccormack2014numerical] and the Jacobian J without giving their discrete form.  Reading R3
(SURVEY O.3): conservative forms built with the same segmented D1 that
differentiates the fluxes, in index space:

  2-D  M_xi = (y_eta, -x_eta),  M_eta = (-y_xi, x_xi),  J^-1 = x_xi y_eta - x_eta y_xi
  3-D  (Thomas-Lombard)  M_{kappa,i} = D_c(x_k D_b x_j) - D_b(x_k D_c x_j)
       for (kappa, b, c) and (i, j, k) cyclic permutations of (0, 1, 2);
       J^-1 = det(d x_i / d kappa) with every entry a D1 of a coordinate.

M[kappa][i] = J^-1 d kappa / d x_i, so grad(kappa) = J M[kappa].  Coordinates are unwrapped
across periodic seams with the mesh's period vectors (x(i+n) = x(i) + period).
Pinned in tests/test_oracle_metrics.py: exact cofactors for quadratic maps, free-stream
preservation sum_kappa D_kappa M[kappa][i] = 0 on hole-free meshes, J^-1 of affine maps.
"""
from __future__ import annotations

import numpy as np

from . import sbp


def axis_of(kappa: int, d: int) -> int:
    """numpy axis of index direction kappa for a spatial array shaped (n_{d-1}, ..., n0)."""
    return d - 1 - kappa


def coordinate_derivatives(xyz, period, positions):
    """dx[c][kappa] = D_kappa x_c (segmented, seam-unwrapped)."""
    d = xyz.shape[0]
    return [[sbp.d1(xyz[c], axis_of(k, d), *positions[k], jump=period[k][c])
             for k in range(d)] for c in range(d)]


def metrics(xyz, period, positions):
    """Returns (Jinv, M) with M[kappa][i] (lists of arrays of the spatial shape)."""
    d = xyz.shape[0]
    dx = coordinate_derivatives(xyz, period, positions)
    if d == 2:
        Jinv = dx[0][0] * dx[1][1] - dx[0][1] * dx[1][0]
        M = [[dx[1][1], -dx[0][1]],
             [-dx[1][0], dx[0][0]]]
        return Jinv, M
    if d != 3:
        raise ValueError("dimension must be 2 or 3")
    M = [[None] * 3 for _ in range(3)]
    for kap in range(3):
        b, c = (kap + 1) % 3, (kap + 2) % 3
        for i in range(3):
            j, k = (i + 1) % 3, (i + 2) % 3
            # D_c(x_k * D_b x_j) - D_b(x_k * D_c x_j)
            t1 = sbp.d1(xyz[k], axis_of(c, 3), *positions[c], jump=period[c][k],
                        factor=dx[j][b])
            t2 = sbp.d1(xyz[k], axis_of(b, 3), *positions[b], jump=period[b][k],
                        factor=dx[j][c])
            M[kap][i] = t1 - t2
    Jinv = (dx[0][0] * (dx[1][1] * dx[2][2] - dx[1][2] * dx[2][1])
            - dx[0][1] * (dx[1][0] * dx[2][2] - dx[1][2] * dx[2][0])
            + dx[0][2] * (dx[1][0] * dx[2][1] - dx[1][1] * dx[2][0]))
    return Jinv, M
