"""Parity at the BASELINE full sizes, in the launch configuration bench.py times.

2-D configs 2 and 3 are small enough for the oracle at full size: setup tables bit-exact,
RHS on every point, and (config 3) the state after the bootstrap and one macro step.  For the
3-D configs 4 and 5 the oracle cannot run whole meshes quickly, so they are checked by
properties that hold at any size (BASELINE north_star): free-stream preservation through
the full MRAB path, and MRAB with every step multiple 1 being bitwise SRAB."""
import numpy as np
import pytest

import synth
from synth.configs import primitive_to_conserved
from oracle import rhs as orhs, timeint
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a_list, b_list):
    num = max(float(np.max(np.abs(a - b))) for a, b in zip(a_list, b_list))
    den = max(float(np.max(np.abs(b))) for b in b_list)
    return num / den


@pytest.fixture(scope="module")
def full3():
    p = synth.make_config(3, "full")
    return p, orhs.build(p)


@pytest.fixture(scope="module")
def full2():
    p = synth.make_config(2, "full")
    return p, orhs.build(p)


@pytest.mark.parametrize("which", ["full2", "full3"])
def test_fullsize_setup_and_rhs(which, request):
    p, st = request.getfixturevalue(which)
    plan = mrab.Plan(p)
    for g in range(len(p.meshes)):
        tb = plan.tables(g)
        rc = st.ov.receivers[g]
        assert np.array_equal(tb["iblank"], st.ov.active[g].ravel().astype(np.int8))
        assert np.array_equal(tb["point"], rc.point)
        assert np.array_equal(tb["donor"], rc.donor)
        assert np.array_equal(tb["base"][:, :p.dim], rc.base)
    ctx = mrab.Context(plan, p.q0)
    rng = np.random.default_rng(7)
    states = [q * (1.0 + 1e-4 * rng.standard_normal(q.shape)) for q in p.q0]
    Rg = ctx.rhs(states)
    Ro = orhs.rhs(p, st, states)
    assert _rel(Rg, Ro) <= 1e-10
    ctx.close()


def test_fullsize_config3_state(full3):
    """Config 3 at full size through the bench's launch path (bootstrap + 1 macro step)."""
    p, st = full3
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    ctx.step(p.history_m - 1 + 1)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    orc = timeint.MRAB(p, setup=st)
    orc.run(1)
    assert _rel(gpu, orc.base) <= 1e-10
    ctx.close()


def _uniform(p, u):
    out = []
    for m in p.meshes:
        shp = tuple(reversed(m.shape))
        vel = [np.full(shp, u)] + [np.zeros(shp)] * (p.dim - 1)
        out.append(primitive_to_conserved(np.ones(shp), vel, np.full(shp, 1 / 1.4)))
    return out


def test_fullsize_config4_free_stream():
    """Uniform flow (equal to the far-field state) is preserved to rounding by the full MRAB
    path on the 24 M-point 3-D config (Cartesian meshes: free stream is exact)."""
    p = synth.make_config(4, "full")
    p.q0 = _uniform(p, 0.3)
    p.q_inf = p.q0[0].reshape(p.nc, -1)[:, 0].copy()
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    ctx.step(p.history_m - 1 + 2)
    for g in range(len(p.meshes)):
        q, _ = ctx.get_state(g)
        assert np.max(np.abs(q - p.q0[g])) <= 1e-12 * np.max(np.abs(p.q0[g]))
    ctx.close()


def test_fullsize_config5_sr1_is_srab():
    """MRAB with every step multiple 1 is single-rate AB: both runs (one through the plan's
    own step multiples forced to 1, one through an explicit all-ones plan) agree bitwise."""
    p = synth.make_config(5, "full", order_n=2)
    G = len(p.meshes)
    a = mrab.Context(mrab.Plan(p, steps=[1] * G), p.q0)
    a.step(p.history_m - 1 + 2)
    for m in p.meshes:
        m.step_multiple = 1
    b = mrab.Context(mrab.Plan(p), p.q0)
    b.step(p.history_m - 1 + 2)
    for g in range(G):
        qa, _ = a.get_state(g)
        qb, _ = b.get_state(g)
        assert np.array_equal(qa, qb)
        assert np.all(np.isfinite(qa))
    a.close()
    b.close()
