"""Space-time convergence pin of the whole oracle (SBP-SAT overset RHS + MRAB): the
convecting vortex of App. C on the box-in-box configuration, third-order
MRAB with step ratio 2.  The paper prints EOC 3.263 / 3.688 / 3.558 (N = 50..200, t = 1);
reading: omega = 2, phi = 8 (not printed), t = 0.25, N = 32/64/128, dt proportional to
the inner spacing."""
import json
import math
import os

import numpy as np
import pytest

from oracle import timeint
from synth.configs import vortex_box_in_box, vortex_exact

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _err(N, T=0.25):
    p = vortex_box_in_box(N)
    p.meshes[0].step_multiple = 2         # outer mesh slow (coarser), inner fast
    dx_in = 0.76 / (N - 1)
    h = 0.3 * dx_in / 3.0
    nmac_total = int(round(T / (2 * h)))
    h = T / (2 * nmac_total)
    p.h = h
    p.order_n = p.history_m = 3
    mr = timeint.MRAB(p)
    mr.run(nmac_total - (p.history_m - 1))
    t = float(mr.t) * h
    assert abs(t - T) < 1e-12
    tot = 0.0
    for g, m in enumerate(p.meshes):
        ex = vortex_exact(m, t)
        act = mr.setup.geom[g].active
        e = (mr.base[g][0] - ex[0])[act]
        hx = m.xyz[0].ravel()[1] - m.xyz[0].ravel()[0]
        hy = m.xyz[1][1, 0] - m.xyz[1][0, 0]
        tot += np.sum(e ** 2) * hx * hy
    return math.sqrt(tot)


@pytest.mark.slow
def test_vortex_space_time_order():
    errs = [_err(N) for N in (32, 64, 128)]
    eoc = math.log(errs[1] / errs[2]) / math.log(2)
    lo, hi = min(GOLD["vortex_eoc"]["values"]), max(GOLD["vortex_eoc"]["values"])
    assert lo - 0.5 < eoc < hi + 0.5, (eoc, errs)
