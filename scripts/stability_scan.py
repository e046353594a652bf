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


N = 13
ONE = 1.0 + 1e-6    # neutral modes (conserved quantities) read 1 + O(1e-9) at eps = 1e-7


def smap_for(h, steps):
    """Step map of the App. C convecting-vortex box-in-box (outer 2 x 1 periodic, inner
    0.76^2, both N x N: spacing ratio 2.6), linearised about the uniform free stream
    rho = 1, u = (0.5, 0), p = 1/gamma with zero histories -- a steady state (P:872-873:
    "starting from a steady-state solution")."""
    p = synth.configs.vortex_box_in_box(N)
    p.order_n, p.history_m, p.h = 3, 3, h
    ctx = mrab.Context(mrab.Plan(p, steps=steps), p.q0)
    ctx.step(p.history_m - 1)
    sm = stability.StepMap(ctx)
    g = p.gamma
    parts = []
    for shp, n in zip(sm.shapes, sm.sizes):
        q = np.empty(shp)
        q[0], q[1], q[2], q[3] = 1.0, 0.5, 0.0, (1.0 / g) / (g - 1.0) + 0.5 * 0.25
        parts.append(q.ravel())
        parts.extend(np.zeros(n) for _ in range(p.history_m - 1))
    return ctx, sm, np.concatenate(parts)


def dense_rho(H, steps):
    c = None
    try:
        c, s, ph = smap_for(H / max(steps), steps)
        return stability.spectral_radius(stability.step_matrix(s, ph))
    except mrab.MrabError:                         # bootstrap or step blew up: unstable
        return float("inf")
    finally:
        if c is not None:
            c.close()


def main():
    out = {"problem": f"vortex box-in-box N={N}, Euler, about the uniform free stream, AB3",
           "eps": stability.EPS, "stable_if_rho_le": ONE, "rho": "dense eigensolve of every eq:sm_form column"}
    Hs = [0.005, 0.01, 0.02, 0.04]
    base = None
    for name, steps in (("srab", [1, 1]), ("mrab_sr2", [2, 1]), ("mrab_sr3", [3, 1])):
        t = time.time()
        row = {"rates": steps, "rho_vs_H": {str(H): dense_rho(H, steps) for H in Hs}}
        row["max_stable_macro_H"] = stability.max_stable(lambda H: dense_rho(H, steps),
                                                         1e-3, 0.1, tol=1e-4, one=ONE)
        row["rho_at_1e-3"] = dense_rho(1e-3, steps)
        if base is None:
            base = row["max_stable_macro_H"]
        row["r_srab"] = row["max_stable_macro_H"] / base
        row["efficiency_pct"] = 100.0 * row["r_srab"] / max(steps)
        row["seconds"] = time.time() - t
        out[name] = row
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
