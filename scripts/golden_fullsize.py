"""Write tests/golden/fullsize_config{4,5}.npz: oracle values of the 3-D configs at their FULL
BASELINE sizes, for tests/test_gpu_fullsize.py (the oracle needs ~1 h per config there, too
long for the GPU suite).  Calls only oracle/ and synth/ (test infrastructure).

Per mesh g:
  * sha256 of the setup tables (iblank int8, receiver points int64, donors int32, stencil
    bases int32 (R, 3)) -- compared bit for bit;
  * the Lagrange weights and metric terms at sampled receivers / points (<= 1e-13);
  * the RHS at q0 on sampled points, and the state after the bootstrap and one MRAB macro
    step on the same points, with the per-component max |.| over the whole mesh (the
    relative bars' denominators).
Samples: 2048 seeded random points, 512 seeded random receivers, and every point within 2
cells of a face or a hole edge along a seeded random line per direction (closures, SAT).
Usage: python scripts/golden_fullsize.py CID [CID ...]
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
import bars  # noqa: E402  (tests/bars.py: the bars' scales, computed with oracle/ only)
from oracle import rhs as orhs, timeint  # noqa: E402

ORDER = {4: 3, 5: 2}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def samples(p, st, g, rng):
    m = p.meshes[g]
    N = m.npts
    rc = st.ov.receivers[g]
    idx = [rng.choice(N, 2048, replace=False)]
    if len(rc.point):
        idx.append(rng.choice(rc.point, min(512, len(rc.point)), replace=False))
    shp = m.shape
    for k in range(3):
        # one random grid line per direction: every active point of it
        fixed = [int(rng.integers(0, shp[a])) for a in range(3)]
        line = []
        for t in range(shp[k]):
            c = list(fixed)
            c[k] = t
            line.append(c[0] + shp[0] * (c[1] + shp[1] * c[2]))
        idx.append(np.array(line, dtype=np.int64))
    return np.unique(np.concatenate(idx))


def main(cid):
    t0 = time.time()
    scale = os.environ.get("GOLDEN_SCALE", "full")          # "test": a dry run of this script
    p = synth.make_config(cid, scale, order_n=ORDER[cid])
    st = orhs.build(p)
    print(f"config {cid}: setup {time.time() - t0:.0f} s", flush=True)
    rng = np.random.default_rng(1234 + cid)
    out = {"order_n": np.array(ORDER[cid]), "G": np.array(len(p.meshes))}
    S = []
    for g, m in enumerate(p.meshes):
        rc = st.ov.receivers[g]
        R = len(rc.point)
        base3 = np.zeros((R, 3), np.int32)
        base3[:, :p.dim] = rc.base
        out[f"m{g}_sha_iblank"] = np.array(sha(st.ov.active[g].ravel().astype(np.int8)))
        out[f"m{g}_sha_point"] = np.array(sha(rc.point.astype(np.int64)))
        out[f"m{g}_sha_donor"] = np.array(sha(rc.donor.astype(np.int32)))
        out[f"m{g}_sha_base"] = np.array(sha(base3))
        out[f"m{g}_nrecv"] = np.array(R)
        rs = np.sort(rng.choice(R, min(2048, R), replace=False)) if R else np.zeros(0, np.int64)
        out[f"m{g}_wsample_rows"] = rs
        out[f"m{g}_wsample"] = rc.weights[rs]
        idx = samples(p, st, g, rng)
        S.append(idx)
        out[f"m{g}_idx"] = idx
        geo = st.geom[g]
        out[f"m{g}_jinv"] = geo.Jinv.ravel()[idx]
        out[f"m{g}_M"] = np.stack([np.stack([geo.M[k][i].ravel()[idx] for i in range(3)]) for k in range(3)])
    t1 = time.time()
    R0 = orhs.rhs(p, st, p.q0)
    print(f"config {cid}: rhs {time.time() - t1:.0f} s", flush=True)
    for g in range(len(p.meshes)):
        Rf = R0[g].reshape(p.nc, -1)
        out[f"m{g}_rhs"] = Rf[:, S[g]]
        out[f"m{g}_rhs_max"] = np.max(np.abs(Rf), axis=1)
    del R0
    out["rhs_scale"] = bars.rhs_scales(p, st, p.q0)
    t2 = time.time()
    orc = timeint.MRAB(p, setup=st)
    orc.run(1)
    print(f"config {cid}: bootstrap + 1 macro step {time.time() - t2:.0f} s", flush=True)
    for g in range(len(p.meshes)):
        Qf = orc.base[g].reshape(p.nc, -1)
        out[f"m{g}_state"] = Qf[:, S[g]]
        out[f"m{g}_state_max"] = np.max(np.abs(Qf), axis=1)
    out["cmax"] = np.array(bars.state_scales(orc.base, p.gamma)[1] / bars.state_scales(orc.base, p.gamma)[0])
    name = f"fullsize_config{cid}.npz" if scale == "full" else f"dryrun_{scale}_config{cid}.npz"
    path = os.path.join(ROOT, "tests", "golden" if scale == "full" else "/tmp", name)
    np.savez_compressed(path, **out)
    print(f"config {cid}: wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB) in {time.time() - t0:.0f} s",
          flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        main(int(a))
