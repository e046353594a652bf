"""Pins of oracle/stability.py (step-matrix procedure; bisection P:877-878).

The step matrix of a linear ODE under AB-n is the companion matrix of the textbook AB
characteristic polynomial z^n - z^(n-1) - h lam sum_k b_k z^k (coefficients typed here, not
taken from oracle/abcoef); the real-axis stability limit of AB3 is h lam = -6/11; a decoupled
two-rate system splits into a fast block applied SR times and a slow AB block of step SR h.
"""
import numpy as np
import pytest

from oracle import stability as stab

AB = {2: [-1 / 2, 3 / 2], 3: [5 / 12, -16 / 12, 23 / 12],
      4: [-9 / 24, 37 / 24, -59 / 24, 55 / 24]}       # oldest first


class _Lin:
    """y_g' = sum_h A[g][h] y_h, one scalar per 'mesh'."""

    def __init__(self, A, n, h, steps):
        self.A = np.asarray(A, dtype=np.float64)
        G = self.A.shape[0]
        self.meshes = [type("M", (), {"step_multiple": s})() for s in steps]
        self.q0 = [np.array([1.0]) for _ in range(G)]
        self.order_n, self.history_m, self.h = n, n, h

    def rhs(self, states, which=None):
        y = np.array([s[0] for s in states])
        d = self.A @ y
        return [np.array([d[g]]) if (which is None or g in which) else None
                for g in range(len(states))]


def _rho_ab(n, z):
    """max |root| of z^n - z^(n-1) - z_h sum_k b_k z^k (b oldest first -> power k)."""
    c = np.zeros(n + 1, dtype=complex)              # highest power first
    c[0] = 1.0
    c[1] = -1.0
    for k, b in enumerate(AB[n]):                   # b_k multiplies z^k
        c[n - k] -= z * b
    return float(np.max(np.abs(np.roots(c))))


def _G(sys_, steps, phi0=None, eps=stab.EPS):
    G = len(steps)
    m = sys_.history_m
    if phi0 is None:
        phi0 = np.random.default_rng(0).standard_normal(G * m)
    return stab.step_matrix(sys_, phi0, eps=eps, steps=steps, rhs_fn=sys_.rhs), phi0


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("hl", [-0.1, -0.3, -0.5, 0.05])
def test_scalar_step_matrix_is_ab_companion(n, hl):
    s = _Lin([[hl / 0.1]], n, 0.1, [1])
    G, _ = _G(s, [1])
    assert G.shape == (n, n)
    assert abs(stab.spectral_radius(G) - _rho_ab(n, hl)) < 1e-6


def test_ab3_real_axis_limit_by_bisection():
    def rho_of(h):
        s = _Lin([[-1.0]], 3, h, [1])
        return stab.spectral_radius(_G(s, [1], eps=1e-6)[0])
    hmax = stab.max_stable(rho_of, 0.1, 1.0, tol=1e-4)
    assert abs(hmax - 6 / 11) < 2e-4


@pytest.mark.parametrize("SR", [2, 3, 4])
def test_decoupled_two_rate(SR):
    """Fast block: AB3 at h applied SR times; slow block: AB3 at SR h (P:569-606 with no
    coupling)."""
    l1, l2, h = -2.0, -0.7, 0.1
    s = _Lin([[l1, 0.0], [0.0, l2]], 3, h, [1, SR])
    G, _ = _G(s, [1, SR])
    exp = max(_rho_ab(3, h * l1) ** SR, _rho_ab(3, SR * h * l2))
    assert abs(stab.spectral_radius(G) - exp) < 1e-6


def test_coupled_map_is_linear_and_eps_independent():
    """For a linear system the macro map is linear: G phi = map(phi) and G does not depend
    on eps (checks the column order and the history packing)."""
    A = [[-1.0, 0.4], [0.3, -0.2]]
    s = _Lin(A, 3, 0.05, [1, 2])
    G7, phi = _G(s, [1, 2])
    G4, _ = _G(s, [1, 2], phi0=phi, eps=1e-4)
    assert np.max(np.abs(G7 - G4)) < 1e-7
    img = stab.macro_map(s, phi, steps=[1, 2], rhs_fn=s.rhs)
    assert np.max(np.abs(G7 @ phi - img)) < 1e-7 * np.max(np.abs(img))


def test_pack_roundtrip():
    st = [np.arange(4.0).reshape(2, 2), np.arange(3.0)]
    H = [[st[0] + 1, st[0] + 2], [st[1] + 1, st[1] + 2]]
    phi = stab.pack(st, H)
    s2, H2 = stab.unpack(phi, [(2, 2), (3,)], 3)
    assert all(np.array_equal(a, b) for a, b in zip(st, s2))
    assert all(np.array_equal(a, b) for x, y in zip(H, H2) for a, b in zip(x, y))
