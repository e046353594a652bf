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


# ---- in_wall_body (R17's wall-body rule) pinned by analytic geometry, not by itself --------
def _wall_mesh(poly):
    """A 2-D mesh whose j = 0 WALL face traces the closed polygon `poly` (n, 2), periodic in i;
    a second radial layer (scaled copy) makes it a valid two-row mesh."""
    poly = np.asarray(poly, dtype=np.float64)
    n = len(poly)
    xyz = np.stack([np.stack([poly[:, 0], 1.5 * poly[:, 0]]), np.stack([poly[:, 1], 1.5 * poly[:, 1]])])
    return synth.configs.Mesh("wall", (n, 2), np.ascontiguousarray(xyz), (True, False),
                              ((synth.PERIODIC, synth.PERIODIC), (synth.WALL, synth.OVERSET)), 1, 1)


@pytest.mark.parametrize("clockwise", [True, False])
def test_in_wall_body_circle(clockwise):
    """The config-3 wall is the 512-gon inscribed in r = 0.5: points with r below the polygon's
    inradius 0.5 cos(pi/512) are inside, points with r > 0.5 outside, for either orientation."""
    n = 512
    th = 2 * np.pi * np.arange(n) / n * (-1 if clockwise else 1)
    m = _wall_mesh(np.stack([0.5 * np.cos(th), 0.5 * np.sin(th)], axis=1))
    rng = np.random.default_rng(1)
    r = rng.uniform(0.0, 1.0, 4000)
    a = rng.uniform(0, 2 * np.pi, 4000)
    X = np.stack([r * np.cos(a), r * np.sin(a)], axis=1)
    ins = overset.in_wall_body(m, X)
    inner = r < 0.5 * np.cos(np.pi / n) - 1e-12
    outer = r > 0.5 + 1e-12
    assert inner.sum() > 500 and outer.sum() > 500
    assert ins[inner].all() and not ins[outer].any()


def test_in_wall_body_nonconvex():
    """An L-shaped wall: the union of [0,2]x[0,1] and [0,1]x[1,2] (exact point classification)."""
    corners = [(0, 0), (2, 0), (2, 1), (1, 1), (1, 2), (0, 2)]
    poly = []
    for a, b in zip(corners, corners[1:] + corners[:1]):      # 8 nodes per unit of edge length
        L = int(round(8 * max(abs(b[0] - a[0]), abs(b[1] - a[1]))))
        for t in range(L):
            poly.append((a[0] + (b[0] - a[0]) * t / L, a[1] + (b[1] - a[1]) * t / L))
    m = _wall_mesh(np.array(poly) - 0.37)          # off-centre so no point sits on a vertex ray
    rng = np.random.default_rng(2)
    X = rng.uniform(-0.5, 2.5, (5000, 2))
    x, y = X[:, 0], X[:, 1]
    inside = ((x > 0) & (x < 2) & (y > 0) & (y < 1)) | ((x > 0) & (x < 1) & (y > 0) & (y < 2))
    d = np.minimum.reduce([np.abs(x), np.abs(y), np.abs(x - 2), np.abs(y - 1), np.abs(x - 1), np.abs(y - 2)])
    clear = d > 1e-9
    assert np.array_equal(overset.in_wall_body(m, X - 0.37)[clear], inside[clear])


def test_config3_hole_against_geometry():
    """Config 3 (test size): background points with r < 0.49 (inside the cylinder body) are holes
    and points with r > 2.2 (outside the O-grid, r in [0.5, 2]) are active; the hole therefore
    lies between the analytic body and the O-grid's outer radius."""
    p = synth.make_config(3, "test")
    ov = overset.build_overset(p.meshes)
    bg = p.meshes[1]
    X = bg.xyz.reshape(2, -1)
    r = np.hypot(X[0], X[1])
    act = ov.active[1].ravel()
    assert not act[r < 0.49].any()
    assert act[r > 2.2].all()
    assert (~act).sum() > (r < 0.49).sum()           # the O-grid cuts beyond the body
