"""Memory-safety tier in place of compute-sanitizer.  The pool refuses
compute-sanitizer ("closed on this pool ... Find a bad access with bounds checks and asserts
of your own, small cases, and a comparison with the CPU reference"), so the same four
questions are asked with the library's own workspace:

* memcheck (writes out of bounds): the workspace sits between two 4 MiB guard bands inside
  one device buffer; every byte of the buffer starts as 0xFF.  After create, bootstrap, MRAB
  steps from the captured graphs, the parity-hook RHS and the accessors, the guard bands are
  still all 0xFF.
* initcheck (reads of never-written memory): the workspace itself starts as 0xFF..FF, a NaN
  in every double.  Any read of an unwritten slot that reaches a result turns it into NaN;
  the states after the steps must be finite and equal to the oracle (per-component bars).
* racecheck / synccheck (shared-memory or stream ordering hazards): two runs are bit for
  bit identical (tests/test_gpu_parity.py::test_run_to_run_bitwise) and the overlapped
  schedule equals the serial one bit for bit (::test_overlapped_schedule_is_bitwise_serial).
Cases span every kernel family: config 1 (2-D Euler, lean + general tiles, donor gather),
config 3 (curvilinear O-grid, wall SAT, critical/bulk split on two streams), config 4 (3-D
two-pass RHS, donor boxes, box-staged gather), config 5 (four rates, curvilinear 3-D)."""
import numpy as np
import pytest

import synth
from bars import assert_states
from oracle import timeint
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GUARD = 4 << 20


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("cid,kw", [(1, {}), (3, {"sr": 4}), (4, {}), (5, {"order_n": 2})])
def test_guard_bands_and_poisoned_workspace(cid, kw):
    p = synth.make_config(cid, "test", **kw)
    plan = mrab.Plan(p)
    nbytes = plan.workspace_bytes()
    buf = torch.full((GUARD + nbytes + 256 + GUARD,), 0xFF, dtype=torch.uint8, device="cuda")
    ws = buf[GUARD:GUARD + nbytes + 256]
    ctx = mrab.Context(plan, p.q0, workspace=ws)
    ctx.step(p.history_m - 1 + 2)
    gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
    R = ctx.rhs(gpu)
    h = ctx.get_history(0, 0)
    ctx.set_history(0, 0, h)
    torch.cuda.synchronize()
    lo = buf[:GUARD]
    # the context uses the first 256-aligned address of ws: bytes before it belong to the band
    base = ws.data_ptr()
    off = (-base) % 256
    hi = buf[GUARD + off + nbytes:]
    assert bool(torch.all(lo == 0xFF)), "write below the workspace"
    assert bool(torch.all(hi == 0xFF)), "write past the end of the workspace"
    for a in gpu + R:
        assert np.all(np.isfinite(a)), "a NaN from a never-written workspace slot"
    orc = timeint.MRAB(p)
    orc.run(2)
    assert_states(gpu, orc.base, p.gamma)
    # round-2 entry points under the same bands: timestep kernel, variable step (tile-list
    # donor preparation), and -- two-rate problems -- a slowest-first context
    dts = ctx.dt()
    assert all(np.isfinite(d) and d > 0 for d in dts)
    ctx.step_h(0.9 * p.s_max * p.h)
    orc.macro_step_var(0.9 * p.s_max * p.h)
    torch.cuda.synchronize()
    assert bool(torch.all(lo == 0xFF)) and bool(torch.all(hi == 0xFF)), "write outside the workspace"
    assert_states([ctx.get_state(g)[0] for g in range(len(p.meshes))], orc.base, p.gamma)
    ctx.close()
    if len({m.step_multiple for m in p.meshes}) == 2 and min(m.step_multiple for m in p.meshes) == 1:
        buf.fill_(0xFF)
        ctx = mrab.Context(plan, p.q0, workspace=ws)
        ctx.step(p.history_m - 1 + 2, scheme="slowest_first_reextrap")
        torch.cuda.synchronize()
        assert bool(torch.all(buf[:GUARD] == 0xFF)) and bool(torch.all(buf[GUARD + off + nbytes:] == 0xFF))
        o2 = timeint.MRAB(p)
        o2.run(2, scheme="slowest_first_reextrap")
        assert_states([ctx.get_state(g)[0] for g in range(len(p.meshes))], o2.base, p.gamma)
        ctx.close()
