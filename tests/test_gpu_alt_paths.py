"""GPU parity of the non-default kernel paths (selected by the MRAB_* switches, read into the
plan's Options at mrab_plan_create; each case runs in a subprocess): the one-pass fused 3-D
RHS (k_rhs3z: z-marching tiles, TMA-staged planes), the per-receiver 3-D gather, the 8^3-tile
divergence pass (k_rhs3d<PRE>; the default is k_div3w on 16 x 8 x 4 tiles), the 3-D task-flow schedule, the 2-D general tile path for every tile (no lean path), and the serial
(non-overlapped) 2-D schedule with uncapped curvilinear tiles.  Each must match the oracle like the
default path (states after N macro steps to 1e-10, RHS to 1e-10)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import synth
from oracle import rhs as orhs, timeint
from paper_1805_06607_b200 import mrab
cid = {cid}
p = synth.make_config(cid, "test")
plan = mrab.Plan(p)
ctx = mrab.Context(plan, p.q0)
st = orhs.build(p)
Rg = ctx.rhs(p.q0)
Ro = orhs.rhs(p, st, p.q0)
rel = max(np.max(np.abs(a - b)) for a, b in zip(Rg, Ro)) / max(np.max(np.abs(b)) for b in Ro)
assert rel <= 1e-10, ("rhs", rel)
ctx.step(p.history_m - 1 + p.n_macro)
gpu = [ctx.get_state(g)[0] for g in range(len(p.meshes))]
orc = timeint.MRAB(p, setup=st)
orc.run(p.n_macro)
rel2 = max(np.max(np.abs(a - b)) for a, b in zip(gpu, orc.base)) / max(np.max(np.abs(b)) for b in orc.base)
assert rel2 <= 1e-10, ("state", rel2)
print("ok", rel, rel2)
"""

CASES = [
    (4, {"MRAB_3D_FUSED": "1"}),
    (5, {"MRAB_3D_FUSED": "1"}),
    (5, {"MRAB_INTERP_BOX": "0"}),
    (4, {"MRAB_DIV_WIDE": "0"}),
    (4, {"MRAB_FLUX_WIDE": "0"}),
    (4, {"MRAB_FLUX_SYM": "0"}),
    (5, {"MRAB_FLUX_WIDE": "0", "MRAB_DIV_WIDE": "0"}),
    (5, {"MRAB_DIV_WIDE": "0"}),
    (5, {"MRAB_OVERLAP3D": "1"}),
    (3, {"MRAB_LEAN": "0"}),
    (3, {"MRAB_TILE_FLAGS": "0"}),
    (2, {"MRAB_OVERLAP": "0", "MRAB_CURV_HALF": "0"}),
]


@pytest.mark.parametrize("cid,env", CASES, ids=[f"cfg{c}-" + "-".join(f"{k}={v}" for k, v in e.items()) for c, e in CASES])
def test_alternative_path_parity(cid, env):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, cid=cid)], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
