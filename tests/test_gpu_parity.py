"""GPU parity: the CUDA path through the C ABI against the oracle (tests/ only may call
oracle/).  Bars (tests/bars.py): states after N macro steps 1e-10 relative
max-norm (BASELINE.json north_star), globally AND per component against the component's
natural scale; RHS 1e-12 per component against the cancellation scale J |D| |Fhat| (and
1e-10 relative max-norm); setup tables bit-exact."""
import numpy as np
import pytest

import synth
from bars import assert_rhs, assert_states
from oracle import rhs as orhs, timeint
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _perturbed(p, seed=11, amp=1e-3):
    rng = np.random.default_rng(seed)
    return [q * (1.0 + amp * rng.standard_normal(q.shape)) for q in p.q0]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mrab.lib()


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_rhs_parity(cid):
    p = synth.make_config(cid, "test")
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    st = orhs.build(p)
    for states in (p.q0, _perturbed(p)):
        Rg = ctx.rhs(states)
        Ro = orhs.rhs(p, st, states)
        rel, pc = assert_rhs(p, st, states, Rg, Ro)
        print(f"config {cid}: rhs rel {rel:.2e}, per component / cancellation scale {pc}")
    ctx.close()


CASES = [(1, {}), (1, {"history_m": 4}), (2, {}), (3, {"sr": 2}), (3, {"sr": 4}),
         (3, {"sr": 8}), (4, {}), (5, {"order_n": 2}), (5, {"order_n": 4})]


@pytest.mark.parametrize("cid,kw", CASES)
def test_state_parity(cid, kw):
    p = synth.make_config(cid, "test", **kw)
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    nboot = p.history_m - 1
    ctx.step(nboot + p.n_macro)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    orc = timeint.MRAB(p)
    orc.run(p.n_macro)
    assert_states(gpu, orc.base, p.gamma)
    ev, point_rhs, mac = ctx.counters()
    # the GPU evaluates R(t) inside the kernel that steps to t + h_g, so the RHS
    # that completes the rings at the end of the oracle's bootstrap is the first evaluation
    # of the GPU's first MRAB macro step, and the GPU's last one is still owed: one fewer
    # evaluation per mesh than the oracle, exactly
    assert list(ev) == [c - 1 for c in orc.counts], (list(ev), orc.counts)
    act_pts = [int(orc.setup.geom[g].active.sum()) for g in range(len(p.meshes))]
    assert point_rhs == sum(a * e for a, e in zip(act_pts, ev))
    assert mac == nboot + p.n_macro
    # holes keep their initial values
    for g in range(len(p.meshes)):
        act = orc.setup.geom[g].active
        assert np.array_equal(gpu[g][:, ~act], p.q0[g][:, ~act])
    ctx.close()


def test_srab_equals_single_rate_run():
    """SRAB (every s_g = 1) on the GPU vs the oracle's single-rate AB."""
    p = synth.make_config(1, "test", n_macro=40)
    plan = mrab.Plan(p, steps=[1, 1])
    ctx = mrab.Context(plan, p.q0)
    ctx.step(p.history_m - 1 + p.n_macro)
    gpu = [ctx.get_state(g)[0] for g in range(2)]
    orc = timeint.MRAB(p, steps=[1, 1])
    orc.run(p.n_macro)
    assert_states(gpu, orc.base, p.gamma)


def test_config1_full_length():
    """Config 1 at its full size and full length (200 slow steps)."""
    p = synth.make_config(1, "full")
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    ctx.step(p.history_m - 1 + p.n_macro)
    gpu = [ctx.get_state(g)[0] for g in range(2)]
    orc = timeint.MRAB(p)
    orc.run(p.n_macro)
    assert_states(gpu, orc.base, p.gamma)


def test_eval_counts():
    p = synth.make_config(2, "test")
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    nboot = p.history_m - 1
    ctx.step(nboot)
    ev0, _, _ = ctx.counters()
    ctx.step(5)
    ev1, pr, _ = ctx.counters()
    d = ev1 - ev0
    assert d[0] == 5 * 1 and d[1] == 5 * 4      # slow bg: 1 per macro step, fast inner: SR


def test_nonfinite_reported():
    """A blown-up state is reported as NONFINITE by mrab_get_state ("rhs blowup")."""
    p = synth.make_config(1, "test")
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    bad = p.q0[1].copy()
    bad[0, 5, 5] = np.nan
    ctx.set_state(1, bad)
    with pytest.raises(mrab.MrabError, match="NONFINITE"):
        ctx.get_state(1)
    q, _ = ctx.get_state(0)
    assert np.all(np.isfinite(q))
    ctx.close()


@pytest.mark.parametrize("cid,kw", [(3, {"sr": 4}), (2, {}), (4, {}), (5, {"order_n": 4}), (5, {"order_n": 2})])
def test_overlapped_schedule_is_bitwise_serial(cid, kw, monkeypatch):
    """The overlapped macro step (2-D: critical/bulk split of the slow mesh on two streams;
    3-D: per-mesh RHS, donor-preparation and gather streams with the donor data of later micro
    indices prepared ahead; node priorities) only reorders independent launches: states equal
    the serial schedule's bit for bit."""
    p = synth.make_config(cid, "test", **kw)
    out = []
    for ov in ("0", "1"):
        monkeypatch.setenv("MRAB_OVERLAP", ov)
        monkeypatch.setenv("MRAB_OVERLAP3D", ov)
        plan = mrab.Plan(p)
        ctx = mrab.Context(plan, p.q0)
        ctx.step(p.history_m - 1 + 6)
        out.append([ctx.get_state(g)[0] for g in range(len(p.meshes))])
        ctx.close()
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cid,size", [(3, "test"), (4, "test"), (3, "full")])
def test_run_to_run_bitwise(cid, size):
    """Two identical runs give bit-identical states: no shared-memory race or ordering hazard in
    the tiled kernels, the gathers or the overlapped schedule changes a single bit (the full-size
    config-3 run exercises the lean interior tiles and the critical/bulk split)."""
    p = synth.make_config(cid, size)
    out = []
    for _ in range(2):
        plan = mrab.Plan(p)
        ctx = mrab.Context(plan, p.q0)
        ctx.step(p.history_m - 1 + 3)
        out.append([ctx.get_state(g)[0] for g in range(len(p.meshes))])
        ctx.close()
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cid", [1, 4])
def test_caller_donor_table_reaches_the_rhs(cid):
    """§8(b): a caller-supplied donor table is what the kernels use.  One receiver's weights
    are changed; the GPU RHS then equals the oracle's RHS with the same change (and differs
    from the unmodified RHS at that receiver)."""
    p = synth.make_config(cid, "test")
    ib, dn = mrab.overset_build(p)
    d2 = dn.copy()
    r = len(dn) // 3
    g = int(d2["recv_mesh"][r])
    d2["w"][r, 0, :] = d2["w"][r, 0, :] + np.array([0.05, -0.02, -0.02, 0.01])
    states = _perturbed(p)
    ctx0 = mrab.Context(mrab.Plan(p), p.q0)
    R0 = ctx0.rhs(states)
    ctx0.close()
    ctx = mrab.Context(mrab.Plan(p, iblank=ib, donors=d2), p.q0)
    Rg = ctx.rhs(states)
    ctx.close()
    st = orhs.build(p)
    rc = st.ov.receivers[g]
    row = int(np.nonzero(rc.point == d2["recv_index"][r])[0][0])
    rc.weights[row] = d2["w"][r][:p.dim]
    st.stencils[g] = orhs._stencils(p, st.ov, g)
    Ro = orhs.rhs(p, st, states)
    assert_rhs(p, st, states, Rg, Ro)
    pt = int(d2["recv_index"][r])
    assert np.max(np.abs(Rg[g].reshape(p.nc, -1)[:, pt] - R0[g].reshape(p.nc, -1)[:, pt])) > 1e-8
