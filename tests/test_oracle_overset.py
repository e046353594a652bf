"""Pins of oracle/overset.py (reading R17 of DESIGN.md)."""
import itertools

import numpy as np
import pytest

from oracle import overset
import synth


def test_lagrange_weights():
    rng = np.random.default_rng(0)
    t = rng.uniform(0, 3, 50)
    W = overset.lagrange_weights(t)
    assert np.allclose(W.sum(axis=1), 1.0, atol=1e-14)
    for deg in range(4):                     # exact for cubic polynomials
        assert np.allclose(W @ (np.arange(4.0) ** deg), t ** deg, atol=1e-12)
    assert np.array_equal(overset.lagrange_weights(np.arange(4.0)), np.eye(4))
    dW = overset.lagrange_dweights(t)
    assert np.allclose(dW @ (np.arange(4.0) ** 3), 3 * t ** 2, atol=1e-11)


def test_shift_order():
    o = overset.shift_order(2)
    assert [tuple(x) for x in o[:5]] == [(0, 0), (0, 1), (0, -1), (1, 0), (-1, 0)]
    assert len(o) == 9


def test_config1_brute_force_pins():
    """SURVEY G17 worked pin (computed there by brute force): background hole = indices
    18..23 in both axes (36 points), 24 hole-edge receivers, 160 inner-face receivers."""
    p = synth.make_config(1)
    ov = overset.build_overset(p.meshes)
    holes = np.argwhere(~ov.active[0])
    assert len(holes) == 36
    assert holes.min(axis=0).tolist() == [18, 18] and holes.max(axis=0).tolist() == [23, 23]
    assert ov.active[1].all()
    assert len(ov.receivers[0].point) == 24 and set(ov.receivers[0].donor) == {1}
    assert len(ov.receivers[1].point) == 160 and set(ov.receivers[1].donor) == {0}


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_donor_invariants(cid):
    """Every receiver is active, its donor stencil is all-active and the stencil's cubic map
    at the donor logical coordinates reproduces the receiver position (brute force); every
    hole is inside a higher-priority mesh or a wall body."""
    p = synth.make_config(cid, "test")
    ov = overset.build_overset(p.meshes)
    for g, m in enumerate(p.meshes):
        rc = ov.receivers[g]
        act = ov.active[g].ravel()
        assert act[rc.point].all()
        X = m.xyz.reshape(m.dim, -1)[:, rc.point].T
        for r in range(len(rc.point)):
            dm = p.meshes[rc.donor[r]]
            st = overset.stencil_flat(dm, rc.base[r])
            assert ov.active[rc.donor[r]].ravel()[st].all()
            offs = np.array(list(itertools.product(range(4), repeat=dm.dim)))[:, ::-1]
            W = np.ones(len(offs))
            for k in range(dm.dim):
                W = W * rc.weights[r, k, offs[:, k]]
            unwrapped = rc.base[r].copy()
            for k in range(dm.dim):      # base of the unwrapped stencil for seam coordinates
                if dm.periodic[k] and rc.xi[r, k] - unwrapped[k] > 3.5:
                    unwrapped[k] += dm.shape[k]
            nodes = overset.node_coords(dm, unwrapped[None, :] + offs)
            scale = np.max(np.abs(np.diff(nodes[:, 0])))
            assert np.allclose(W @ nodes, X[r], atol=1e-10 * max(1.0, scale))
        holes = np.nonzero(~act)[0]
        if len(holes):
            Xh = m.xyz.reshape(m.dim, -1)[:, holes].T
            ins = np.zeros(len(holes), bool)
            for B, mb in enumerate(p.meshes):
                if B != g and mb.priority > m.priority:
                    ins |= np.all(np.isfinite(overset.find_cells(mb, Xh)), axis=1)
                if B != g:
                    ins |= overset.in_wall_body(mb, Xh)
            assert ins.all()
