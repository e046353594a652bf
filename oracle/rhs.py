"""The coupled SBP-SAT right-hand side of all overset meshes (ORACLE, test infrastructure).

For every mesh g (eq:int; App. C; readings R3, R11-R19 of DESIGN.md):
  1. primitives rho, u, p, T                                                      (R12)
  2. viscous only: d_kappa phi by segmented D1 for phi in (u_1..u_d, T), Cartesian
     gradients d_i phi = J sum_kappa M[kappa][i] D_kappa phi                      (R3/O.4)
  3. Cartesian fluxes F^I_i and F^V_i                                             (R11)
  4. contravariant fluxes Fhat_kappa = sum_i M[kappa][i] (F^I_i - F^V_i)
  5. R = -J sum_kappa D_kappa Fhat_kappa at active points, 0 at holes
  6. SAT at every segment end (kappa, side) facing a hole, an overset face or a physical
     face (P:279-299, P:292-294 edge/corner rule):
        R += -(1/p0) [sigma_I K^side(grad kappa; q) + sigma1_V I] (q - qhat)
             + (1/p0) sigma2_side (F^V_kappa - Fhat^V_kappa)
     sigma_I = 1/2, sigma1_V = |grad kappa|^2 / (2 Re), sigma2_+- = +-1/2, p0 = 17/48,
     side + = kappa-min end, - = kappa-max end, F^V_kappa = sum_i (grad kappa)_i F^V_i.
        interface : qhat = Lagrange interpolation of the donor state, Fhat^V_kappa =
                    sum_i (grad kappa)_i * (interpolated donor Cartesian F^V_i)    (R18)
        far field : qhat = q_inf, Fhat^V = 0                                        (R16)
        wall      : qhat = (rho, 0, rho T_w/(gamma(gamma-1))), sigma2 term dropped  (R16)
Interpolation uses the donor mesh's state at the same evaluation time (R8).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from . import gas, metrics, overset, sbp

P0 = float(sbp.H_BOUNDARY[0])         # p0 = H_00 = 17/48 (R14)
SIGMA_I = 0.5
INTERFACE = overset.OVERSET


@dataclass
class MeshGeom:
    Jinv: np.ndarray
    J: np.ndarray
    M: list
    active: np.ndarray
    positions: list
    sat: list            # list of (flat points, kappa, side, type) groups


@dataclass
class Setup:
    problem: object
    ov: overset.OversetSetup
    geom: List[MeshGeom]
    recv_row: List[dict]
    stencils: list = None


def _sat_groups(mesh, positions):
    d = mesh.dim
    groups = []
    for k in range(d):
        a, b = positions[k]
        ax = d - 1 - k
        n = mesh.shape[k]
        idx = np.arange(n).reshape([n if i == ax else 1 for i in range(d)])
        for side, pos, face_idx, bc in ((+1, a, 0, mesh.face_bc[k][0]),
                                         (-1, b, n - 1, mesh.face_bc[k][1])):
            end = pos == 0
            if mesh.periodic[k]:
                groups.append((np.nonzero(end.ravel())[0], k, side, INTERFACE))
                continue
            at_face = np.broadcast_to(idx == face_idx, end.shape)
            groups.append((np.nonzero((end & ~at_face).ravel())[0], k, side, INTERFACE))
            groups.append((np.nonzero((end & at_face).ravel())[0], k, side, bc))
    return [g for g in groups if len(g[0])]


def build(problem) -> Setup:
    ov = overset.build_overset(problem.meshes)
    geom = []
    for g, m in enumerate(problem.meshes):
        Jinv, M = metrics.metrics(m.xyz, m.period, ov.positions[g])
        act = ov.active[g]
        if np.any(Jinv[act] <= 0):
            raise ValueError(f"mesh {g}: non-positive J^-1 at an active point")
        J = np.where(act, 1.0 / np.where(act, Jinv, 1.0), 0.0)
        geom.append(MeshGeom(Jinv, J, M, act, ov.positions[g], _sat_groups(m, ov.positions[g])))
    recv_row = [{int(p): r for r, p in enumerate(rc.point)} for rc in ov.receivers]
    stencils = [_stencils(problem, ov, g) for g in range(len(problem.meshes))]
    return Setup(problem, ov, geom, recv_row, stencils)


def _gradients(prob, geo, q):
    d = prob.dim
    rho, u, p, T = gas.primitives(q, prob.gamma)
    fields = list(u) + [T]
    Dphi = [[sbp.d1(phi, metrics.axis_of(k, d), *geo.positions[k]) for k in range(d)]
            for phi in fields]
    grad = [[geo.J * sum(geo.M[k][i] * Dphi[f][k] for k in range(d)) for i in range(d)]
            for f in range(len(fields))]
    du = [grad[i] for i in range(d)]          # du[i][j] = d u_i / d x_j
    dT = grad[d]
    return du, dT


def cartesian_viscous_fluxes(prob, setup, g, q):
    """[F^V_i for i < d], each (nc, *spatial); zeros for inviscid problems."""
    d = prob.dim
    if not prob.viscous:
        return [np.zeros_like(q) for _ in range(d)]
    du, dT = _gradients(prob, setup.geom[g], q)
    return [gas.viscous_flux(q, du, dT, i, prob.Re, prob.Pr, prob.gamma) for i in range(d)]


def _stencils(problem, ov, g):
    """Per receiver of mesh g: flat donor stencil indices (R, 4^d) and tensor-product
    Lagrange weights (R, 4^d)."""
    rc = ov.receivers[g]
    d = problem.dim
    offs = overset._stencil_offsets(d)
    R = len(rc.point)
    idx = np.zeros((R, 4 ** d), dtype=np.int64)
    W = np.ones((R, 4 ** d))
    for r in range(R):
        idx[r] = overset.stencil_flat(problem.meshes[rc.donor[r]], rc.base[r])
    for k in range(d):
        W = W * rc.weights[:, k, :][:, offs[:, k]]
    return idx, W


def interpolate(setup, g, fields_per_mesh):
    """Lagrange interpolation of per-mesh arrays (C, *spatial) at the receivers
    of mesh g: qhat_r = sum_a W_ra f_donor(r)[stencil_ra]; returns (R, C)."""
    rc = setup.ov.receivers[g]
    idx, W = setup.stencils[g]
    C_ = fields_per_mesh[0].shape[0]
    out = np.zeros((len(rc.point), C_))
    for dm in np.unique(rc.donor):
        sel = rc.donor == dm
        F = fields_per_mesh[dm].reshape(C_, -1)
        out[sel] = np.einsum("rca,ra->rc", F[:, idx[sel]].transpose(1, 0, 2), W[sel])
    return out


def contravariant_fluxes(problem, geo, q, FV):
    """Fhat_kappa = sum_i M[kappa][i] (F^I_i - F^V_i), kappa < d (step 4)."""
    d = problem.dim
    FI = [gas.inviscid_flux(q, i, problem.gamma) for i in range(d)]
    return [sum(geo.M[k][i][None] * (FI[i] - FV[i]) for i in range(d)) for k in range(d)]


def interior_rhs(problem, geo, q, FV):
    """R = -J sum_kappa D_kappa Fhat_kappa on active points, 0 at holes (steps 4-5)."""
    d = problem.dim
    R = np.zeros_like(q)
    for k, Fhat in enumerate(contravariant_fluxes(problem, geo, q, FV)):
        for c in range(d + 2):
            R[c] += sbp.d1(Fhat[c], metrics.axis_of(k, d), *geo.positions[k])
    R = -geo.J[None] * R
    R[:, ~geo.active] = 0.0
    return R


def rhs(problem, setup: Setup, states, which=None):
    """Coupled RHS at the given states (list of (nc, *spatial) arrays) of the meshes in
    `which` (default all; the others get None).  Donor data always come from all meshes."""
    d = problem.dim
    nc = d + 2
    G = len(problem.meshes)
    FV = [cartesian_viscous_fluxes(problem, setup, g, states[g]) for g in range(G)]
    FVstack = [np.concatenate(FV[g], axis=0) for g in range(G)]    # (d*nc, *spatial)
    out = []
    for g in range(G):
        if which is not None and g not in which:
            out.append(None)
            continue
        geo = setup.geom[g]
        q = states[g]
        R = interior_rhs(problem, geo, q, FV[g])
        # ---- SAT -------------------------------------------------------------------
        qhat_i = interpolate(setup, g, states)
        fvhat_i = interpolate(setup, g, FVstack) if problem.viscous else None
        Rf = R.reshape(nc, -1)
        qf = q.reshape(nc, -1)
        for pts, k, side, typ in geo.sat:
            qp = qf[:, pts].T                                     # (P, nc)
            n = np.stack([(geo.J * geo.M[k][i]).ravel()[pts] for i in range(d)], axis=1)
            if typ == INTERFACE:
                rows = np.searchsorted(setup.ov.receivers[g].point, pts)
                qh = qhat_i[rows]
            elif typ == overset.FARFIELD:
                qh = np.broadcast_to(problem.q_inf, qp.shape)
            elif typ == overset.WALL:
                qh = np.zeros_like(qp)
                qh[:, 0] = qp[:, 0]
                qh[:, -1] = qp[:, 0] * problem.wall_T / (problem.gamma * (problem.gamma - 1))
            else:
                raise ValueError("periodic faces carry no SAT")
            K = gas.k_matrix(qp, n, side, problem.gamma)
            dq = qp - qh
            pen = SIGMA_I * np.einsum("pij,pj->pi", K, dq)
            if problem.viscous:
                sig1 = np.sum(n * n, axis=1) / (2.0 * problem.Re)
                pen = pen + sig1[:, None] * dq
            sat = -pen / P0
            if problem.viscous and typ != overset.WALL:
                fvk = sum(n[:, i][:, None] * FV[g][i].reshape(nc, -1)[:, pts].T
                          for i in range(d))
                if typ == INTERFACE:
                    fvh = sum(n[:, i][:, None] * fvhat_i[rows][:, i * nc:(i + 1) * nc]
                              for i in range(d))
                else:
                    fvh = 0.0
                sat = sat + (0.5 * side) * (fvk - fvh) / P0
            Rf[:, pts] += sat.T
        out.append(R)
    return out
