"""Host logic of the GPU stability laboratory without a GPU: StepMap's integrator-vector
layout (state, then m-1 history entries oldest first, mesh by mesh) against a fake context,
and the bisection helper."""
import numpy as np

from paper_1805_06607_b200 import stability


class _FakePlan:
    nc, history_m, n_meshes = 2, 3, 2
    shapes = [(3, 2), (2, 2)]                      # (ni, nj): arrays are [nc][nj][ni]


class _FakeCtx:
    """Stores state/history; step(1) applies the linear map y -> 2y, H_k -> H_k + k."""

    def __init__(self):
        self.plan = _FakePlan()
        rng = np.random.default_rng(1)
        self.q = [rng.standard_normal((2, 2, 3)), rng.standard_normal((2, 2, 2))]
        self.H = [[rng.standard_normal(q.shape) for _ in range(2)] for q in self.q]

    def get_state(self, g):
        return self.q[g].copy(), 0.0

    def set_state(self, g, src):
        self.q[g] = src.copy()

    def get_history(self, g, k):
        return self.H[g][k].copy()

    def set_history(self, g, k, src):
        self.H[g][k] = src.copy()

    def step(self, n):
        self.q = [2 * q for q in self.q]
        self.H = [[h + k for k, h in enumerate(Hg)] for Hg in self.H]


def test_stepmap_layout_and_columns():
    ctx = _FakeCtx()
    sm = stability.StepMap(ctx)
    assert sm.dim == (12 + 8) * 3
    phi = sm.read()
    exp = np.concatenate([ctx.q[0].ravel(), ctx.H[0][0].ravel(), ctx.H[0][1].ravel(),
                          ctx.q[1].ravel(), ctx.H[1][0].ravel(), ctx.H[1][1].ravel()])
    assert np.array_equal(phi, exp)
    G = stability.step_matrix(sm, phi, eps=1e-3)
    d = np.ones(sm.dim)
    for o in (0, 36):                               # state blocks of mesh 0 / mesh 1
        n = 12 if o == 0 else 8
        d[o:o + n] = 2.0
    assert np.allclose(G, np.diag(d), atol=1e-9)
    assert abs(stability.spectral_radius(G) - 2.0) < 1e-9


def test_max_stable_bisection():
    x = stability.max_stable(lambda h: 1.0 + (h - 0.3), 0.0, 1.0, tol=1e-6)
    assert abs(x - 0.3) < 1e-6
    assert stability.max_stable(lambda h: 0.5, 0.0, 1.0) == 1.0


def test_krylov_and_power_match_dense_on_fake_linear_map():
    ctx = _FakeCtx()
    sm = stability.StepMap(ctx)
    phi = sm.read()
    assert abs(stability.spectral_radius_krylov(sm, phi, eps=1e-3, tol=1e-10) - 2.0) < 1e-6
    assert abs(stability.power_estimate(sm, phi, iters=40, eps=1e-3) - 2.0) < 1e-6


def test_arnoldi_uses_converged_ritz_values_only():
    """Explicitly restarted Arnoldi on a fake non-normal linear step map: an isolated unstable
    eigenvalue is found to 1e-6; with a stable spectrum clustered below 1 the estimate stays
    below 1 (unconverged Ritz values, which can leave the spectrum of a non-normal matrix, are
    not used)."""
    from paper_1805_06607_b200 import stability as gs
    rng = np.random.default_rng(1)
    n = 400
    lam = np.concatenate([1 - 0.2 * rng.random(n - 1) ** 3, [-1.004]])
    X = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    Xi = np.linalg.inv(X)
    phi0 = rng.standard_normal(n)
    A = X @ np.diag(lam) @ Xi
    rho, _ = gs.spectral_radius_arnoldi(lambda p: A @ p, phi0, k=60)
    assert abs(rho - 1.004) <= 1e-6
    lam[-1] = -0.99
    A2 = X @ np.diag(lam) @ Xi
    rho, _ = gs.spectral_radius_arnoldi(lambda p: A2 @ p, phi0, k=60)
    assert rho <= 1.0
