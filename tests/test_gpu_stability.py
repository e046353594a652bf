"""GPU step-matrix stability procedure against the oracle's (tests/ only call
oracle/).  Tiny overset problem: the inviscid box-in-box of App. C at N = 17 (4440-element
integrator vector: 2 meshes x 4 components x (state + 2 history entries)), AB3, rates 2:1.
Tolerances: the map itself 1e-10 relative (north_star); step-matrix columns formed with
eps = 1e-5 so that the finite-difference rounding noise (~1e-13 |phi| / eps) stays below the
1e-6 bar; the power-iteration estimate of rho to 1e-6 relative."""
import numpy as np
import pytest

import synth
from oracle import rhs as orhs, stability as ostab
from paper_1805_06607_b200 import mrab, stability

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
STEPS = [2, 1]


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = synth.configs.mms_box_in_box(17, "inviscid")
    p.order_n, p.history_m, p.h = 3, 3, 0.002
    ctx = mrab.Context(mrab.Plan(p, steps=STEPS), p.q0)
    with pytest.raises(mrab.MrabError, match="INSUFFICIENT_HISTORY"):
        ctx.get_history(0, 0)
    ctx.step(p.history_m - 1)                      # bootstrap
    smap = stability.StepMap(ctx)
    phi0 = smap.read()
    yield p, orhs.build(p), smap, phi0
    ctx.close()


def _omap(p, st):
    return lambda phi: ostab.macro_map(p, phi, steps=STEPS, setup=st)


def test_map_parity(setup):
    p, st, smap, phi0 = setup
    assert phi0.size == smap.dim == 4 * (17 * 17 + 9 * 9) * 3
    g = smap(phi0)
    o = _omap(p, st)(phi0)
    assert np.max(np.abs(g - o)) <= 1e-10 * np.max(np.abs(o))
    # history entries round-trip through set/get unchanged
    smap.write(phi0)
    assert np.array_equal(smap.read(), phi0)


def test_step_matrix_columns(setup):
    p, st, smap, phi0 = setup
    rng = np.random.default_rng(5)
    n1 = 4 * 17 * 17
    # state and both history entries of each mesh
    cols = sorted(set(rng.integers(0, phi0.size, 16).tolist()
                      + [0, n1 - 1, n1, 2 * n1, 3 * n1, 3 * n1 + 4 * 81, phi0.size - 1]))
    Gg = stability.step_matrix(smap, phi0, eps=1e-5, cols=cols)
    om = _omap(p, st)
    base = om(phi0)
    for c, j in enumerate(cols):
        ph = phi0.copy()
        ph[j] += 1e-5
        col = (om(ph) - base) / 1e-5
        assert np.max(np.abs(Gg[:, c] - col)) <= 1e-6 * max(1.0, np.max(np.abs(col))), j


def test_power_estimate_parity(setup):
    p, st, smap, phi0 = setup
    rg = stability.power_estimate(smap, phi0, iters=20, eps=1e-5, seed=3)
    om = _omap(p, st)
    base = om(phi0)
    v = np.random.default_rng(3).standard_normal(phi0.size)
    v /= np.linalg.norm(v)
    for _ in range(20):
        w = (om(phi0 + 1e-5 * v) - base) / 1e-5
        ro = float(np.linalg.norm(w))
        v = w / ro
    assert abs(rg - ro) <= 1e-6 * ro, (rg, ro)
    print(f"rho estimate gpu {rg:.9f} oracle {ro:.9f}")


def test_history_accessor_errors(setup):
    p, st, smap, phi0 = setup
    ctx = smap.ctx
    for k in (-1, p.history_m - 1):
        with pytest.raises(mrab.MrabError, match="INVALID"):
            ctx.get_history(0, k)
    buf = np.zeros(16)
    assert mrab.lib().mrab_get_history(ctx.h, 2, 0, buf.ctypes.data) == 1    # MRAB_E_INVALID
    assert mrab.lib().mrab_get_history(ctx.h, 0, 0, None) == 1


def test_rk_step_matches_oracle_rk4_and_heun():
    """mrab_rk_step (the reference integrator of the stability tables) against the
    oracle's rk_step on the coupled SBP-SAT RHS: 3 steps of RK4 and of Heun's RK3."""
    import synth
    from oracle import rhs as orhs, timeint
    p = synth.make_config(1, "test")
    st = orhs.build(p)
    rhs_fn = lambda s, which=None: orhs.rhs(p, st, s, which)  # noqa: E731
    for order in (4, 3):
        ctx = mrab.Context(mrab.Plan(p), p.q0)
        h = 2.5 * p.h
        ctx.rk_step(h, 3, order)
        y = [q.copy() for q in p.q0]
        for _ in range(3):
            y = timeint.rk_step(rhs_fn, y, h, timeint.rk_tableau(order))
        for g in range(len(p.meshes)):
            q = ctx.get_state(g)[0]
            assert np.max(np.abs(q - y[g])) <= 1e-12 * np.max(np.abs(y[g]))
        ctx.close()


def test_arnoldi_matches_dense_rho():
    """Restarted Arnoldi on the matrix-free step map against the dense eigensolve of every
    eq:sm_form column (13 x 13 App. C box-in-box, rates 2:1, AB3)."""
    from paper_1805_06607_b200 import stability as gs
    p = synth.configs.vortex_box_in_box(9)
    p.order_n, p.history_m, p.h = 3, 3, 0.004
    ctx = mrab.Context(mrab.Plan(p, steps=[2, 1]), p.q0)
    ctx.step(p.history_m - 1)
    sm = gs.StepMap(ctx)
    phi = sm.read()
    dense = gs.spectral_radius(gs.step_matrix(sm, phi))
    arn, nmv = gs.spectral_radius_arnoldi(sm, phi, k=80, restarts=8)
    # only converged Ritz values count, so the estimate never exceeds the spectrum; it equals
    # rho when the leading eigenvalue has converged
    gr = gs.growth_rate(sm, phi, iters=300)
    print("dense", dense, "arnoldi", arn, nmv, "power", gr)
    assert arn <= dense * (1 + 1e-5), (arn, dense, nmv)
    assert dense - 5e-3 <= gr <= dense * (1 + 2e-4), (gr, dense)
    ctx.close()


def test_device_resident_step_matrix_equals_host(setup):
    """step_matrix_device keeps every integrator vector on the GPU (device-to-device accessor
    copies, differences in torch): its columns equal the host-round-trip ones to the last bit or
    two (torch divides by eps through a reciprocal multiply; the stepped vectors are identical)."""
    p, st, smap, phi0 = setup
    cols = [0, 7, 300, 1111, 2222, 4439]
    Gh = stability.step_matrix(smap, phi0, cols=cols)
    Gd = stability.step_matrix_device(smap, phi0, cols=cols).cpu().numpy()
    assert np.allclose(Gh, Gd, rtol=5e-16, atol=0.0)
