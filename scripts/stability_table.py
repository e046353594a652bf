"""Stability table in the format of Table t:thirdstab on synthetic config 1 (the
2-D overset vortex pair: background 41^2, h 0.25, slow; inner 41^2, h 0.0625, fast; spacing
ratio 4), on the GPU path: for RK4, SRAB and MRAB with SR = 2..8, AB3 and AB34, the maximum
stable macro step (bisection to 1e-4) of the step matrix (eq:sm / eq:sm_form,
eps = 1e-7) linearised about the uniform free stream (a steady state of the discretisation),
rho from converged Arnoldi Ritz values and the power-iteration growth of the matrix-free step map, and r_RK4, r_SRAB, % = r_SRAB / SR.
Prints markdown and one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_1805_06607_b200 import mrab, stability  # noqa: E402

ONE = 1.0 + 2e-4          # growth per step above this = unstable: d rho / d H ~ 1/H here, so the
                          # 1e-4 bisection of H needs rho resolved to ~1e-3; neutral
                          # modes read 1 + O(1e-9) through eq:sm_form (DESIGN.md R-SM)
ITERS = int(os.environ.get("POWER_ITERS", "300"))


def rho_est(smap, phi):
    """max(converged Arnoldi eigenvalue, asymptotic power-iteration growth)."""
    g = stability.growth_rate(smap, phi, iters=ITERS)
    if not np.isfinite(g) or g > 1.5:
        return g
    a, _ = stability.spectral_radius_arnoldi(smap, phi, k=K, restarts=2)
    return max(a, g)
SCALE = os.environ.get("SCALE", "full")
CFG = int(os.environ.get("CFG", "1"))                 # 1: Euler vortex pair; 2: viscous curvilinear pair
TOL = float(os.environ.get("TOL", "1e-4"))            # bisection tolerance (1e-4)
LO = float(os.environ.get("LO", "1e-3"))
K = int(os.environ.get("ARNOLDI_K", "70"))


def problem(order_n, history_m, sr):
    p = synth.make_config(CFG, SCALE, order_n=order_n, history_m=history_m, sr=sr)
    # steady base state: the far-field state everywhere
    q = [np.broadcast_to(np.asarray(p.q_inf).reshape((-1,) + (1,) * p.dim), x.shape).copy() for x in p.q0]
    p.q0 = q
    return p


def rho_mrab(H, order_n, history_m, sr):
    p = problem(order_n, history_m, sr)
    p.h = H / sr
    ctx = None
    try:
        ctx = mrab.Context(mrab.Plan(p), p.q0)
        ctx.step(p.history_m - 1)
        sm = stability.StepMap(ctx)
        parts = []
        for g, n in enumerate(sm.sizes):
            parts.append(p.q0[g].ravel())
            parts.extend(np.zeros(n) for _ in range(p.history_m - 1))
        return rho_est(sm, np.concatenate(parts))
    except mrab.MrabError:
        return float("inf")
    finally:
        if ctx is not None:
            ctx.close()


def rho_rk4(dt):
    p = problem(3, 3, 1)
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    try:
        rm = stability.RKMap(ctx, dt, 4)
        return rho_est(rm, np.concatenate([q.ravel() for q in p.q0]))
    except mrab.MrabError:
        return float("inf")
    finally:
        ctx.close()


def main():
    srs = [int(x) for x in os.environ.get("SRS", "1,2,3,4,5,6,8").split(",")]
    hi = float(os.environ.get("HI", "0.6"))
    t0 = time.time()
    out = {"problem": f"config {CFG} ({SCALE}), about the uniform free stream", "eps": stability.EPS,
           "stable_if_rho_le": ONE, "rho": f"max(converged Ritz value of restarted Arnoldi k = {K}, power-iteration growth over {ITERS} steps)", "bisection_tol": TOL}
    dt_rk4 = stability.max_stable(rho_rk4, LO, hi, tol=TOL, one=ONE)
    out["rk4"] = dt_rk4
    rows = {}
    for name, (n, m) in (("AB3", (3, 3)), ("AB34", (3, 4))):
        base = None
        rows[name] = []
        for sr in srs:
            dt = stability.max_stable(lambda H: rho_mrab(H, n, m, sr), LO, hi, tol=TOL, one=ONE)
            if sr == 1:
                base = dt
            rows[name].append({"sr": sr, "dt": dt, "r_rk4": dt / dt_rk4, "r_srab": dt / base,
                               "pct": 100.0 * dt / base / sr})
            print(name, rows[name][-1], f"{time.time() - t0:.0f} s", flush=True)
    out["rows"] = rows
    out["seconds"] = time.time() - t0
    print("| Int. | SR | dt (AB3) | r_RK4 | r_SRAB | % | dt (AB34) | r_RK4 | r_SRAB | % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    print(f"| RK4 | | {dt_rk4:.5f} | 1.000 | {dt_rk4 / rows['AB3'][0]['dt']:.2f} | | {dt_rk4:.5f} | 1.000 | "
          f"{dt_rk4 / rows['AB34'][0]['dt']:.2f} | |")
    for a, b in zip(rows["AB3"], rows["AB34"]):
        nm = "SRAB" if a["sr"] == 1 else "MRAB"
        print(f"| {nm} | {a['sr']} | {a['dt']:.5f} | {a['r_rk4']:.3f} | {a['r_srab']:.2f} | {a['pct']:.1f} | "
              f"{b['dt']:.5f} | {b['r_rk4']:.3f} | {b['r_srab']:.2f} | {b['pct']:.1f} |")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
