"""Gas model, fluxes and the SAT characteristic matrices (ORACLE, test infrastructure).

Conserved variables q = (rho, rho u_1..rho u_d, rho E).  Equations in strong
conservation form, App. C:
    F^I_i = (rho u_i, rho u_i u_j + p delta_ij, (rho E + p) u_i)
    F^V_i = (0, tau_ij, u_j tau_ij - q_i)
Readings: R11 constant mu = 1, Stokes lambda = -2/3 mu, tau scaled by 1/Re,
Fourier heat flux q_i = -mu/(Re Pr (gamma-1)) d_i T; R12 nondimensionalisation
rho_inf = 1, p_inf = 1/gamma, c_inf = 1, T = gamma p / rho (so c^2 = T),
rho E = p/(gamma-1) + rho|u|^2/2.

K^+- of eq:int = T diag((|Lambda| +- Lambda)/2) T^-1 for the Euler flux Jacobian
A(n) = sum_i n_i dF^I_i/dq at the receiver's own state (reading R15).  Here A(n) is formed
by complex-step differentiation of `inviscid_flux` (exact to rounding) and T, Lambda by a
numerical eigen-decomposition — deliberately not the analytic characteristic formulas the
CUDA path uses.  Pinned in tests/test_oracle_gas.py: K+ - K- = A, K+ K- = 0, spectrum of
A = {u.n (d-fold), u.n +- c|n|}, 1-D reduction.
"""
from __future__ import annotations

import numpy as np


def primitives(q, gamma):
    d = q.shape[0] - 2
    rho = q[0]
    u = [q[1 + i] / rho for i in range(d)]
    ke = 0.5 * rho * sum(ui * ui for ui in u)
    p = (gamma - 1.0) * (q[d + 1] - ke)
    T = gamma * p / rho
    return rho, u, p, T


def inviscid_flux(q, i, gamma):
    """F^I_i (first-derivative terms)."""
    d = q.shape[0] - 2
    rho, u, p, T = primitives(q, gamma)
    comps = [q[1 + i]]
    for j in range(d):
        comps.append(q[1 + j] * u[i] + (p if i == j else 0.0))
    comps.append((q[d + 1] + p) * u[i])
    return np.stack(comps)


def stress(du, Re):
    """tau_ij = (mu/Re)(d_j u_i + d_i u_j) + (lambda/Re) div(u) delta_ij, mu = 1,
    lambda = -2/3 (P:1559-1561 with reading R11).  du[i][j] = d u_i / d x_j."""
    d = len(du)
    div = sum(du[k][k] for k in range(d))
    return [[(du[i][j] + du[j][i] - (2.0 / 3.0) * div * (1.0 if i == j else 0.0)) / Re
             for j in range(d)] for i in range(d)]


def viscous_flux(q, du, dT, i, Re, Pr, gamma):
    """F^V_i = (0, tau_ij, u_j tau_ij - q_i), q_i = -mu/(Re Pr (gamma-1)) d_i T (R11)."""
    d = q.shape[0] - 2
    rho, u, p, T = primitives(q, gamma)
    tau = stress(du, Re)
    heat = -dT[i] / (Re * Pr * (gamma - 1.0))
    comps = [np.zeros_like(rho)]
    for j in range(d):
        comps.append(tau[i][j])
    comps.append(sum(u[j] * tau[i][j] for j in range(d)) - heat)
    return np.stack(comps)


def flux_jacobian(q, n, gamma, eps=1e-30):
    """A(n) = sum_i n_i dF^I_i/dq by complex step.  q: (P, nc), n: (P, d) -> (P, nc, nc)."""
    q = np.asarray(q, dtype=np.float64)
    P, nc = q.shape
    d = nc - 2
    A = np.zeros((P, nc, nc))
    for j in range(nc):
        qc = q.astype(np.complex128)
        qc[:, j] += 1j * eps
        Fn = sum(n[:, i][None, :] * inviscid_flux(qc.T, i, gamma) for i in range(d))
        A[:, :, j] = Fn.T.imag / eps
    return A


def k_matrix(q, n, side, gamma):
    """K^side(n; q) = T diag(max(side*lambda, 0)) T^-1 (readings R14/R15).

    Evaluated as the matrix function f(A), f(lambda) = max(side*lambda, 0), of the
    complex-step Jacobian A(n) by Sylvester's formula over the three distinct eigenvalues
    of the Euler Jacobian, u.n (d-fold), u.n +- c|n| (textbook closed form; always distinct
    since c|n| > 0):  f(A) = sum_k f(lambda_k) prod_{j != k} (A - lambda_j I)/(lambda_k -
    lambda_j).  This equals T f(Lambda) T^-1 for the diagonalisable A without forming T.
    side = +1 (kappa-min face) or -1 (kappa-max face), scalar or per point."""
    q = np.asarray(q, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    A = flux_jacobian(q, n, gamma)
    P, nc = q.shape
    d = nc - 2
    rho, u, p, T = primitives(q.T, gamma)
    un = sum(u[i] * n[:, i] for i in range(d))
    cn = np.sqrt(T) * np.sqrt(np.sum(n * n, axis=1))
    lams = [un, un + cn, un - cn]
    side = np.broadcast_to(np.asarray(side, dtype=np.float64), (P,))
    I = np.eye(nc)[None]
    K = np.zeros((P, nc, nc))
    for k in range(3):
        proj = np.broadcast_to(I, (P, nc, nc)).copy()
        for j in range(3):
            if j != k:
                proj = proj @ ((A - lams[j][:, None, None] * I)
                               / (lams[k] - lams[j])[:, None, None])
        K += np.maximum(side * lams[k], 0.0)[:, None, None] * proj
    return K
