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
