"""Pins of oracle/gas.py: flux homogeneity, the Euler spectrum, K+- identities,
viscous stress of linear fields."""
import numpy as np
import pytest

from oracle import gas

G = 1.4


def _random_states(rng, P, d):
    rho = rng.uniform(0.5, 2.0, P)
    u = rng.uniform(-0.8, 0.8, (d, P))
    p = rng.uniform(0.3, 1.5, P)
    q = np.zeros((d + 2, P))
    q[0] = rho
    q[1:1 + d] = rho * u
    q[d + 1] = p / (G - 1) + 0.5 * rho * np.sum(u * u, axis=0)
    return q, rho, u, p


@pytest.mark.parametrize("d", [1, 2, 3])
def test_flux_homogeneous_degree_one(d):
    """Euler fluxes are homogeneous of degree 1: A(n) q = F_n(q) (independent of T, Lambda)."""
    rng = np.random.default_rng(d)
    q, rho, u, p = _random_states(rng, 20, d)
    n = rng.standard_normal((20, d))
    A = gas.flux_jacobian(q.T, n, G)
    Fn = sum(n[:, i][None] * gas.inviscid_flux(q, i, G) for i in range(d))
    assert np.allclose(np.einsum("pij,jp->ip", A, q), Fn, atol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_k_matrices(d):
    rng = np.random.default_rng(10 + d)
    q, rho, u, p = _random_states(rng, 16, d)
    n = rng.standard_normal((16, d))
    A = gas.flux_jacobian(q.T, n, G)
    Kp = gas.k_matrix(q.T, n, +1, G)
    Km = gas.k_matrix(q.T, n, -1, G)
    assert np.allclose(Kp - Km, A, atol=1e-11)            # (|L|+L)/2 - (|L|-L)/2 = L
    assert np.allclose(Kp @ Km, 0.0, atol=1e-10)
    c = np.sqrt(G * p / rho)
    un = np.sum(u * n.T, axis=0)
    nn = np.linalg.norm(n, axis=1)
    for P in range(16):
        ev = np.sort(np.linalg.eigvals(A[P]).real)
        expect = np.sort([un[P]] * d + [un[P] + c[P] * nn[P], un[P] - c[P] * nn[P]])
        assert np.allclose(ev, expect, atol=1e-10)
        assert np.all(np.linalg.eigvals(Kp[P]).real > -1e-10)


def test_k_one_dimensional_reduction():
    """For supersonic flow in +x every characteristic enters a kappa-min face: K+ = A, K- = 0."""
    q, rho, u, p = _random_states(np.random.default_rng(3), 4, 2)
    q[1] = rho * 3.0
    q[2] = 0.0
    q[3] = p / (G - 1) + 0.5 * rho * 9.0
    n = np.tile([[1.0, 0.0]], (4, 1))
    A = gas.flux_jacobian(q.T, n, G)
    assert np.allclose(gas.k_matrix(q.T, n, +1, G), A, atol=1e-11)
    assert np.allclose(gas.k_matrix(q.T, n, -1, G), 0.0, atol=1e-11)


def test_viscous_flux_linear_field():
    """Linear velocity u = (a y, 0): tau_12 = a/Re, tau_11 = 0; energy flux u_j tau_ij - q_i."""
    Re, Pr = 50.0, 0.72
    q = np.array([[1.0], [0.3], [0.0], [2.0]])
    du = [[np.array([0.0]), np.array([2.0])], [np.array([0.0]), np.array([0.0])]]
    dT = [np.array([0.5]), np.array([0.0])]
    Fx = gas.viscous_flux(q, du, dT, 0, Re, Pr, G)
    Fy = gas.viscous_flux(q, du, dT, 1, Re, Pr, G)
    assert np.allclose(Fx[:, 0], [0, 0, 2 / Re, 0.3 * 0 + 0.5 / (Re * Pr * (G - 1))])
    assert np.allclose(Fy[:, 0], [0, 2 / Re, 0, 0.3 * 2 / Re])
    # divergence-free trace: tau_ii with div u = 3 gives (2 - 2/3*... ) check stokes
    du2 = [[np.array([1.0]), np.array([0.0])], [np.array([0.0]), np.array([2.0])]]
    tau = gas.stress(du2, 1.0)
    assert np.isclose(tau[0][0][0], 2 * 1 - 2 / 3 * 3) and np.isclose(tau[1][1][0], 4 - 2)
