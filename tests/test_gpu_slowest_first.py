"""SURVEY §8(f) f3 on the GPU path: the two-rate slowest-first MRAB variants (P:536-548,
reading R-SF) against the oracle's macro_step_sf, on 2-D Euler, 2-D curvilinear viscous,
the wall-bounded O-grid pair and the 3-D pair."""
import numpy as np
import pytest

import synth
from bars import assert_states
from oracle import rhs as orhs, timeint
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("scheme", ["slowest_first", "slowest_first_reextrap"])
@pytest.mark.parametrize("cid,kw", [(1, {}), (1, {"order_n": 3, "history_m": 4}), (2, {}), (3, {"sr": 2}), (4, {})])
def test_slowest_first_state_parity(cid, kw, scheme):
    p = synth.make_config(cid, "test", **kw)
    st = orhs.build(p)
    nmac = 4
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    ctx.step(p.history_m - 1 + nmac, scheme=scheme)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    ev = ctx.counters()[0] if hasattr(ctx, "counters") else None
    orc = timeint.MRAB(p, setup=st)
    orc.run(nmac, scheme=scheme)
    assert_states(gpu, orc.base, p.gamma)
    if ev is not None:
        # the GPU defers the fast meshes' last evaluation to the next macro step
        for g, m in enumerate(p.meshes):
            assert ev[g] == orc.counts[g] - (1 if m.step_multiple == 1 else 0)
    # and the schemes are distinguishable at this tolerance on a coupled problem
    ctx2 = mrab.Context(mrab.Plan(p), p.q0)
    ctx2.step(p.history_m - 1 + nmac)
    ff = [ctx2.get_state(g)[0] for g in range(len(p.meshes))]
    assert max(np.max(np.abs(a - b)) for a, b in zip(gpu, ff)) > 0.0
    ctx.close()
    ctx2.close()


def test_scheme_errors():
    p = synth.make_config(5, "test", order_n=2)     # four rates
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    with pytest.raises(mrab.MrabError):
        ctx.step(1, scheme="slowest_first")
    ctx.close()
    p = synth.make_config(1, "test")
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    ctx.step(p.history_m - 1 + 1)                   # fastest-first from here on
    with pytest.raises(mrab.MrabError):
        ctx.step(1, scheme="slowest_first")
    ctx.close()
