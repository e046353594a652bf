"""CPU-side checks of the C ABI: the library loads, exports every symbol include/mrab.h
declares, its AB weights match the exact rationals, and its host setup (hole cutting,
receivers, donor stencils, weights, metrics) matches the oracle bit-exactly / to 1e-13."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from oracle import abcoef, rhs as orhs
from paper_1805_06607_b200 import mrab

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mrab.h")).read()
    declared = set(re.findall(r"\b(mrab_[a-z_]+)\s*\(", hdr))
    lib = ctypes.CDLL(mrab.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(mrab.EXPORTED)


@pytest.mark.parametrize("m,n", [(2, 2), (3, 3), (4, 3), (4, 4), (5, 4)])
def test_ab_weights_vs_rationals(m, n):
    nodes = [-(m - 1) + k for k in range(m)]
    for b in (0.25, 0.5, 1.0):
        got = mrab.ab_weights(nodes, n, 0.0, b)
        exp = [float(x) for x in abcoef.ab_weights(nodes, n, 0, b)]
        assert np.allclose(got, exp, rtol=0, atol=1e-15)


def test_ab_weights_errors():
    with pytest.raises(mrab.MrabError, match="INSUFFICIENT_HISTORY"):
        mrab.ab_weights([0.0, 1.0], 3, 0, 1)
    with pytest.raises(mrab.MrabError, match="DEGENERATE_NODES"):
        mrab.ab_weights([0.0, 0.0, 1.0], 3, 0, 1)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_setup_tables_bit_exact(cid):
    p = synth.make_config(cid, "test")
    plan = mrab.Plan(p)
    st = orhs.build(p)
    for g in range(len(p.meshes)):
        tb = plan.tables(g)
        rc = st.ov.receivers[g]
        assert np.array_equal(tb["iblank"], st.ov.active[g].ravel().astype(np.int8))
        assert np.array_equal(tb["point"], rc.point)
        assert np.array_equal(tb["donor"], rc.donor)
        assert np.array_equal(tb["base"][:, :p.dim], rc.base)
        if len(rc.point):
            assert np.max(np.abs(tb["weights"][:, :p.dim] - rc.weights)) < 1e-13
        jinv, M = plan.metrics(g)
        geo = st.geom[g]
        scale = np.max(np.abs(geo.Jinv))
        assert np.max(np.abs(jinv - geo.Jinv.ravel())) <= 1e-13 * scale
        for k in range(p.dim):
            for i in range(p.dim):
                sc = max(np.max(np.abs(geo.M[k][k])), 1e-300)
                assert np.max(np.abs(M[k, i] - geo.M[k][i].ravel())) <= 1e-13 * sc


def test_plan_errors():
    p = synth.make_config(1, "test")
    p.history_m = 2
    with pytest.raises(mrab.MrabError, match="INSUFFICIENT_HISTORY"):
        mrab.Plan(p)
    p = synth.make_config(1, "test")
    p.meshes[0].step_multiple = 3          # 3 does not divide... 3 is the max; make 2 & 3
    p.meshes[1].step_multiple = 2
    with pytest.raises(mrab.MrabError, match="MISALIGNED"):
        mrab.Plan(p)
    p = synth.make_config(1, "test")
    p.meshes[1].xyz = np.ascontiguousarray(p.meshes[1].xyz[:, :, ::-1])   # left-handed
    with pytest.raises(mrab.MrabError):
        mrab.Plan(p)


def test_product_path_is_independent_of_the_oracle():
    """The package (CUDA binding, stability laboratory) never imports oracle/, and the oracle
    never imports the package (the two share no code)."""
    pkg = os.path.join(ROOT, "paper_1805_06607_b200")
    for d, pat in ((pkg, r"^\s*(from|import)\s+oracle\b"),
                   (os.path.join(ROOT, "oracle"), r"^\s*(from|import)\s+paper_1805_06607_b200\b")):
        for f in os.listdir(d):
            if f.endswith(".py"):
                src = open(os.path.join(d, f)).read()
                assert not re.search(pat, src, re.M), f


def _plan_tables(plan, G):
    return [plan.tables(g) for g in range(G)]


@pytest.mark.parametrize("cid", [1, 3, 4, 5])
def test_caller_supplied_setup_reproduces_built_plan(cid):
    """mrab_overset_build exports the blanking and donor table; feeding them (and the plan's
    metric terms) back through mrab_mesh_desc.iblank / .metrics and mrab_problem.donors gives
    a plan whose tables and metrics equal the library-built ones bit for bit (§8(b))."""
    p = synth.make_config(cid, "test")
    G = len(p.meshes)
    ref = mrab.Plan(p)
    ib, dn = mrab.overset_build(p)
    tb = _plan_tables(ref, G)
    assert len(dn) == sum(len(t["point"]) for t in tb)
    for g in range(G):
        assert np.array_equal(ib[g], tb[g]["iblank"])
        sel = dn[dn["recv_mesh"] == g]
        assert np.array_equal(sel["recv_index"], tb[g]["point"])
        assert np.array_equal(sel["donor_mesh"], tb[g]["donor"])
        assert np.array_equal(sel["base"], tb[g]["base"])
        assert np.array_equal(sel["w"], tb[g]["weights"])
    mets = []
    for g in range(G):
        jinv, M = ref.metrics(g)
        mets.append(np.concatenate([jinv[None], M.reshape(p.dim * p.dim, -1)]))
    for kw in (dict(iblank=ib), dict(donors=dn, iblank=ib), dict(metrics=mets),
               dict(iblank=ib, donors=dn, metrics=mets)):
        pl = mrab.Plan(p, **kw)
        for g, t in enumerate(_plan_tables(pl, G)):
            for key in ("iblank", "point", "donor", "base", "weights"):
                assert np.array_equal(t[key], tb[g][key]), (kw.keys(), g, key)
            j1, M1 = pl.metrics(g)
            j0, M0 = ref.metrics(g)
            assert np.array_equal(j1, j0) and np.array_equal(M1, M0)
            assert np.array_equal(pl.face_flags(g), ref.face_flags(g))


@pytest.mark.parametrize("cid", [1, 3, 4])
def test_face_flags_match_oracle_sat_faces(cid):
    """mrab_plan_get_face_flags against the oracle's SAT groups (eq:int): bit 2k =
    side + (kappa-min end), bit 2k+1 = side - (kappa-max end), bit for bit."""
    p = synth.make_config(cid, "test")
    plan = mrab.Plan(p)
    st = orhs.build(p)
    for g in range(len(p.meshes)):
        want = np.zeros(int(np.prod(p.meshes[g].shape[:p.dim])), np.uint8)
        for pts, k, side, _typ in st.geom[g].sat:
            want[pts] |= np.uint8(1 << (2 * k + (0 if side > 0 else 1)))
        assert np.array_equal(plan.face_flags(g), want)


def test_caller_supplied_setup_errors():
    p = synth.make_config(1, "test")
    ib, dn = mrab.overset_build(p)
    with pytest.raises(mrab.MrabError, match="ORPHAN"):
        mrab.Plan(p, iblank=ib, donors=dn[1:])                  # a receiver without a donor
    d2 = dn.copy()
    d2["recv_index"][0] = 0 if dn["recv_index"][0] != 0 else 1  # not a receiver
    d2 = np.concatenate([d2, dn[:1]])
    with pytest.raises(mrab.MrabError, match="INVALID"):
        mrab.Plan(p, iblank=ib, donors=d2)
    d3 = np.concatenate([dn, dn[:1]])                           # duplicate
    with pytest.raises(mrab.MrabError, match="INVALID"):
        mrab.Plan(p, iblank=ib, donors=d3)
    d4 = dn.copy()
    d4["donor_mesh"][0] = d4["recv_mesh"][0]                    # self-donation
    with pytest.raises(mrab.MrabError, match="INVALID"):
        mrab.Plan(p, iblank=ib, donors=d4)
    # a donor stencil over the background's hole
    d5 = dn.copy()
    r = int(np.nonzero(dn["donor_mesh"] == 0)[0][0])
    d5["base"][r, :2] = [19, 19]
    with pytest.raises(mrab.MrabError, match="INVALID"):
        mrab.Plan(p, iblank=ib, donors=d5)
    mets = []
    for g in range(2):
        jinv, M = mrab.Plan(p).metrics(g)
        mets.append(np.concatenate([jinv[None], M.reshape(4, -1)]))
    mets[1][0, 7] = -1.0                                        # J^-1 <= 0
    with pytest.raises(mrab.MrabError, match="INVALID"):
        mrab.Plan(p, metrics=mets)
    ib2 = [b.copy() for b in ib]
    n0, n1 = p.meshes[1].shape[:2]
    ib2[1][n0 * (n1 // 2) + 4] = 0                              # leaves a 4-point segment
    with pytest.raises(mrab.MrabError, match="SEGMENT"):
        mrab.Plan(p, iblank=ib2)
