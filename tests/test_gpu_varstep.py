"""SURVEY §8(f) f2 on the GPU path: the on-device timestep estimate (K9, eq:ts P:620-643) and
the variable macro step (per-step weights from the actual history node times),
against the oracle."""
import math

import numpy as np
import pytest

import synth
from bars import assert_states
from oracle import rhs as orhs, timeint, timestep
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_dt_kernel_matches_oracle(cid):
    """Per-mesh min of eq:ts at q0 and after a few steps: <= 1e-13 relative (the reduction is
    exact; the per-point arithmetic differs by rounding order only)."""
    p = synth.make_config(cid, "test")
    st = orhs.build(p)
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    want = timestep.dt_min(p, st, p.q0)
    got = ctx.dt()
    for a, b in zip(got, want):
        assert abs(a - b) <= 1e-13 * b, (got, want)
    ctx.step(p.history_m - 1 + 2)
    states = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    want = timestep.dt_min(p, st, states)
    got = ctx.dt()
    for a, b in zip(got, want):
        assert abs(a - b) <= 1e-13 * b, (got, want)
    ctx.close()


@pytest.mark.parametrize("cid,kw", [(1, {}), (1, {"order_n": 3, "history_m": 4}), (2, {}), (4, {}),
                                    (5, {"order_n": 4}), (5, {"order_n": 2})])
def test_variable_macro_step_state_parity(cid, kw):
    """Bootstrap, then macro steps H_i = H (1 + 0.3 sin(1.7 i)) (and one fixed-step call in
    between, which must take the variable path too): states vs the oracle's macro_step_var."""
    p = synth.make_config(cid, "test", **kw)
    st = orhs.build(p)
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    orc = timeint.MRAB(p, setup=st)
    ctx.step(p.history_m - 1)
    orc.bootstrap()
    H0 = p.s_max * p.h
    for i in range(5):
        H = H0 * (1.0 + 0.3 * math.sin(1.7 * i))
        if i == 3:
            ctx.step(1)
            orc.macro_step()
        else:
            ctx.step_h(H)
            orc.macro_step_var(H)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    assert_states(gpu, orc.base, p.gamma)
    t = ctx.get_state(0)[1]
    assert abs(t - float(orc.time)) <= 1e-12 * float(orc.time)
    ctx.close()


def test_constant_H_equals_fixed_step():
    """mrab_step_h with H = S h follows mrab_step (graphs, tabulated weights) to rounding."""
    p = synth.make_config(1, "test")
    out = []
    for var in (False, True):
        ctx = mrab.Context(mrab.Plan(p), p.q0)
        ctx.step(p.history_m - 1)
        if var:
            ctx.step_h(p.s_max * p.h, 6)
        else:
            ctx.step(6)
        out.append([ctx.get_state(g)[0] for g in range(len(p.meshes))])
        ctx.close()
    for a, b in zip(*out):
        assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))


def test_cfl_driven_run():
    """The loop a user runs: H from the device estimate every step (CFL 0.5), same on the
    oracle side with its own estimate."""
    p = synth.make_config(2, "test")
    st = orhs.build(p)
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    orc = timeint.MRAB(p, setup=st)
    ctx.step(p.history_m - 1)
    orc.bootstrap()
    S = p.s_max
    for i in range(4):
        Hg = 0.5 * S * min(d / m.step_multiple for d, m in zip(ctx.dt(), p.meshes))
        Ho = timestep.macro_step(p, st, orc.base, 0.5)
        assert abs(Hg - Ho) <= 1e-12 * Ho
        ctx.step_h(Ho)
        orc.macro_step_var(Ho)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    assert_states(gpu, orc.base, p.gamma)
    ctx.close()


def test_step_cfl_matches_manual_loop():
    """mrab_step_cfl = mrab_dt + the H formula + mrab_step_h, bit for bit."""
    p = synth.make_config(1, "test")
    S = p.s_max
    a = mrab.Context(mrab.Plan(p), p.q0)
    b = mrab.Context(mrab.Plan(p), p.q0)
    a.step(p.history_m - 1)
    b.step(p.history_m - 1)
    for _ in range(3):
        H = 0.4 * S * min(d / m.step_multiple for d, m in zip(a.dt(), p.meshes))
        a.step_h(H)
    Hb = b.step_cfl(0.4, 3)
    assert Hb == H
    for g in range(2):
        assert np.array_equal(a.get_state(g)[0], b.get_state(g)[0])
    a.close()
    b.close()


def test_step_h_errors():
    p = synth.make_config(1, "test")
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    with pytest.raises(mrab.MrabError):
        ctx.step_h(p.s_max * p.h)          # bootstrap not done
    ctx.step(p.history_m - 1)
    with pytest.raises(mrab.MrabError):
        ctx.step_h(-1.0)
    ctx.close()
