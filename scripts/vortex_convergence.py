"""Space-time convergence of the whole GPU path on the paper's convecting-vortex test
(App. C, Table t:mms1): box-in-box, outer [-1,1] x [-0.5,0.5] periodic, inner
[-0.38,0.38]^2, both N x N, u0 = 2, error in density at t = 1 in the discrete L2 norm, third-order
MRAB with step ratio 2 (outer mesh slow) and single-rate AB3.  The vortex strength and width
are not printed (reading: omega = 2, phi = 8), so the error levels are not
comparable with the table, the orders are (printed EOC 3.263 / 3.688 / 3.558)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1805_06607_b200 import mrab  # noqa: E402
from synth.configs import vortex_box_in_box, vortex_exact  # noqa: E402


def err(N, sr, T=1.0):
    p = vortex_box_in_box(N)
    p.meshes[0].step_multiple = sr
    dx_in = 0.76 / (N - 1)
    h = 0.3 * dx_in / 3.0
    nmac = int(round(T / (sr * h)))
    p.h = T / (sr * nmac)
    p.order_n = p.history_m = 3
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    ctx.step(nmac)
    tot = 0.0
    for g, m in enumerate(p.meshes):
        q, t = ctx.get_state(g)
        assert abs(t - T) < 1e-9
        ex = vortex_exact(m, T)
        act = plan.tables(g)["iblank"].reshape(q[0].shape) != 0
        e = (q[0] - ex[0])[act]
        hx = m.xyz[0].ravel()[1] - m.xyz[0].ravel()[0]
        hy = m.xyz[1][1, 0] - m.xyz[1][0, 0]
        tot += np.sum(e ** 2) * hx * hy
    ctx.close()
    return math.sqrt(tot)


def main():
    Ns = [int(x) for x in os.environ.get("NS", "50,100,150,200").split(",")]
    out = {}
    for name, sr in (("MRAB SR 2", 2), ("SRAB", 1)):
        es = [err(N, sr) for N in Ns]
        eoc = [None] + [math.log(es[i - 1] / es[i]) / math.log(Ns[i] / Ns[i - 1]) for i in range(1, len(Ns))]
        out[name] = {"N": Ns, "log10_err": [math.log10(e) for e in es], "eoc": eoc}
        print(f"{name}: | N | log10 ||eps||_2 | EOC |")
        for N, e, o in zip(Ns, es, eoc):
            print(f"| {N} | {math.log10(e):.4f} | {'-' if o is None else f'{o:.3f}'} |")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
