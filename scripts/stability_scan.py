"""Step-matrix stability laboratory on the GPU: rho(G_eps) of one MRAB macro
step for the tiny inviscid box-in-box (App. C, N = 17), dense (every column, eq:sm_form) at
one h, and the max stable macro step by bisection on the power-iteration estimate for SRAB
(rates 1:1) and MRAB (rates 2:1).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_1805_06607_b200 import mrab, stability  # noqa: E402


def smap_for(h, steps, N=17):
    p = synth.configs.mms_box_in_box(N, "inviscid")
    p.order_n, p.history_m, p.h = 3, 3, h
    ctx = mrab.Context(mrab.Plan(p, steps=steps), p.q0)
    ctx.step(p.history_m - 1)
    sm = stability.StepMap(ctx)
    return ctx, sm, sm.read()


def main():
    out = {"problem": "mms box-in-box inviscid N=17, AB3", "eps": stability.EPS}
    ctx, sm, phi = smap_for(0.002, [2, 1])
    t = time.time()
    G = stability.step_matrix(sm, phi)
    tG = time.time() - t
    out["dense"] = {"h": 0.002, "rates": [2, 1], "dim": int(phi.size),
                    "rho": stability.spectral_radius(G), "columns_s": tG}
    ctx.close()
    print(json.dumps(out), flush=True)
    for name, steps in (("srab", [1, 1]), ("mrab_sr2", [2, 1])):
        def rho_of(H):
            c = None
            try:
                c, s, ph = smap_for(H / max(steps), steps)
                return stability.power_estimate(s, ph, iters=60)
            except mrab.MrabError:                 # bootstrap or step blew up: unstable
                return float("inf")
            finally:
                if c is not None:
                    c.close()
        Hmax = stability.max_stable(rho_of, 0.001, 0.2, tol=1e-4)
        out[name] = {"rates": steps, "max_stable_macro_H": Hmax,
                     "max_stable_micro_h": Hmax / max(steps)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
