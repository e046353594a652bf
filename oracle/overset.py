"""Overset (Chimera) setup: hole cutting, receivers, donor search, Lagrange weights
(ORACLE, test infrastructure).

PAPER.md §2.2 lists the phases -- bounding-box collision, hole cutting / fringe
determination, donor-receiver pair search, Lagrange interpolation of donor data with
"weights determined as a function of Lagrange shape functions" -- and defers the algorithms
to [bodony2011provably].  The deterministic rules below are reading R17 of
DESIGN.md §2:

 * inside(A, B): an A-point is inside mesh B if some cell of B contains it, i.e. Newton on
   the tensor-cubic Lagrange map of that cell's 4^d stencil converges to logical
   coordinates inside the cell (start at the cell centre, stop when |delta xi| <= 1e-12,
   at most 50 iterations, abandon beyond 4 cells).  Candidate cells: those whose corner-node bounding box,
   grown by 10 % of its extent + 1e-9, contains the point; tried in increasing flat cell
   index (i fastest); the first accepted wins.  Logical coordinates within 1e-12 of an
   integer are snapped to it.
 * hole(A) = (A-points inside any higher-priority mesh, or inside a wall body)
             minus the union of A's donor stencils of the overset-FACE points of the other
             meshes.
 * receivers: active points that end a segment (in any direction) next to a hole or an
   overset face.
 * donor of a receiver: the other meshes in decreasing priority (ties: mesh order); in the
   first one containing the point, stencil base s = floor(xi) - 1 (clamped to [0, n-4], or
   wrapped on periodic directions); if the 4^d stencil is not all-active, shifts
   delta in {0,+1,-1}^d are tried by sum|delta| ascending, then lexicographically with axis 0
   most significant and 0 < +1 < -1.  No all-active stencil anywhere -> orphan (error).
 * weights w_a(t) = prod_{b != a} (t - b)/(a - b), a, b in {0..3}, t = xi - s, per axis.
Pinned in tests/test_oracle_overset.py: weights sum to 1, reproduce tensor polynomials of
degree <= 3, one-hot on nodes; brute-force receiver/hole pins on config 1 (hole = indices
18..23, 24 hole-edge + 160 face receivers).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import List

import numpy as np

from . import sbp

SNAP = 1e-12
NEWTON_TOL = 1e-12          # |delta xi| in logical (cell) units
NEWTON_MAXIT = 50
BBOX_GROW = 0.1
BBOX_ABS = 1e-9

OVERSET, FARFIELD, WALL, PERIODIC = 0, 1, 2, 3


class OrphanReceiver(RuntimeError):
    pass


class SegmentTooShort(RuntimeError):
    pass


# -------------------------------------------------------------------------------------
# Lagrange basis on the nodes 0, 1, 2, 3
# -------------------------------------------------------------------------------------
def lagrange_weights(t):
    t = np.asarray(t, dtype=np.float64)
    out = []
    for a in range(4):
        w = np.ones_like(t)
        for b in range(4):
            if b != a:
                w = w * (t - b) / (a - b)
        out.append(w)
    return np.stack(out, axis=-1)


def lagrange_dweights(t):
    t = np.asarray(t, dtype=np.float64)
    out = []
    for a in range(4):
        acc = np.zeros_like(t)
        for c in range(4):
            if c == a:
                continue
            term = np.full_like(t, 1.0 / (a - c))
            for b in range(4):
                if b != a and b != c:
                    term = term * (t - b) / (a - b)
            acc = acc + term
        out.append(acc)
    return np.stack(out, axis=-1)


# -------------------------------------------------------------------------------------
# geometry helpers
# -------------------------------------------------------------------------------------
def flat_index(shape, idx):
    """idx (..., d) in index order -> flat index (i fastest)."""
    f = np.zeros(idx.shape[:-1], dtype=np.int64)
    stride = 1
    for k in range(len(shape)):
        f = f + idx[..., k] * stride
        stride *= shape[k]
    return f


def node_coords(mesh, idx):
    """Coordinates of nodes idx (..., d) (periodic indices may leave [0, n); the seam is
    unwrapped with the period vectors)."""
    d = mesh.dim
    idx = np.asarray(idx, dtype=np.int64)
    wrapped = idx.copy()
    shift = np.zeros(idx.shape[:-1] + (d,))
    for k in range(d):
        n = mesh.shape[k]
        if mesh.periodic[k]:
            w = np.floor_divide(idx[..., k], n)
            wrapped[..., k] = idx[..., k] - w * n
            shift = shift + w[..., None] * np.asarray(mesh.period[k])[None]
    flat = flat_index(mesh.shape, wrapped)
    X = mesh.xyz.reshape(d, -1)[:, flat]
    return np.moveaxis(X, 0, -1) + shift


def _cells(mesh):
    """All cell lower corners (ncell, d), flat cell order (i fastest)."""
    ranges = [np.arange(mesh.shape[k] if mesh.periodic[k] else mesh.shape[k] - 1)
              for k in range(mesh.dim)]
    grids = np.meshgrid(*reversed(ranges), indexing="ij")
    return np.stack([g.ravel() for g in reversed(grids)], axis=-1)


BLOCK = 8      # cells per axis of the coarse bounding-box blocks (a pure pre-filter)


def cell_bboxes(mesh):
    """Grown corner-node bounding boxes of every cell (flat cell order), plus a coarse level:
    the cells grouped by index-space blocks of BLOCK^d cells with the union box of each block.
    The blocks only pre-filter candidate cells; the candidates are re-sorted into flat cell
    order, so the cells tried (and the first accepted) are exactly those of the flat scan."""
    cells = _cells(mesh)
    corners = np.array(list(itertools.product([0, 1], repeat=mesh.dim)))
    lo = np.full((len(cells), mesh.dim), np.inf)
    hi = np.full((len(cells), mesh.dim), -np.inf)
    for c in corners:                                               # one corner at a time
        P = node_coords(mesh, cells + c[None])
        lo = np.minimum(lo, P)
        hi = np.maximum(hi, P)
    g = BBOX_GROW * (hi - lo) + BBOX_ABS
    lo, hi = lo - g, hi + g
    nb = [-(-(mesh.shape[k] if mesh.periodic[k] else mesh.shape[k] - 1) // BLOCK) for k in range(mesh.dim)]
    bid = np.zeros(len(cells), dtype=np.int64)
    stride = 1
    for k in range(mesh.dim):
        bid += (cells[:, k] // BLOCK) * stride
        stride *= nb[k]
    order = np.argsort(bid, kind="stable")
    starts = np.concatenate([[0], np.nonzero(np.diff(bid[order]))[0] + 1])
    blo = np.minimum.reduceat(lo[order], starts, axis=0)
    bhi = np.maximum.reduceat(hi[order], starts, axis=0)
    ends = np.concatenate([starts[1:], [len(order)]])
    return cells, lo, hi, (order, starts, ends, blo, bhi)


def stencil_base_from_cell(mesh, c):
    """Base of the 4^d Newton stencil for cell c (unwrapped)."""
    s = np.asarray(c, dtype=np.int64) - 1
    for k in range(mesh.dim):
        if not mesh.periodic[k]:
            s[..., k] = np.clip(s[..., k], 0, mesh.shape[k] - 4)
    return s


def _stencil_offsets(d):
    return np.array(list(itertools.product(range(4), repeat=d)))[:, ::-1]   # (4^d, d) i fastest


def cubic_map(mesh, base, xi):
    """X(xi) and dX/dxi of the tensor-cubic Lagrange map of the stencil at `base`.
    base, xi: (P, d).  Returns X (P, d), Jac (P, d, d) with Jac[:, c, k] = dX_c/dxi_k."""
    d = mesh.dim
    offs = _stencil_offsets(d)
    nodes = node_coords(mesh, base[:, None, :] + offs[None])          # (P, 4^d, d)
    t = xi - base
    W = lagrange_weights(t)                                           # (P, d, 4)
    dW = lagrange_dweights(t)
    wprod = np.ones((len(xi), len(offs)))
    for k in range(d):
        wprod = wprod * W[:, k, :][:, offs[:, k]]
    X = np.einsum("pa,pac->pc", wprod, nodes)
    Jac = np.zeros((len(xi), d, d))
    for k in range(d):
        g = np.ones((len(xi), len(offs)))
        for l in range(d):
            g = g * (dW if l == k else W)[:, l, :][:, offs[:, l]]
        Jac[:, :, k] = np.einsum("pa,pac->pc", g, nodes)
    return X, Jac


def _newton(mesh, X, cells):
    """Newton for logical coordinates of points X (P, d) in cells (P, d).  Returns xi
    (P, d) and an accept mask."""
    base = stencil_base_from_cell(mesh, cells)
    xi = cells.astype(np.float64) + 0.5
    conv = np.zeros(len(X), dtype=bool)
    alive = np.ones(len(X), dtype=bool)
    for _ in range(NEWTON_MAXIT):
        idx = np.nonzero(alive & ~conv)[0]
        if len(idx) == 0:
            break
        Xm, Jm = cubic_map(mesh, base[idx], xi[idx])
        try:
            delta = np.linalg.solve(Jm, (X[idx] - Xm)[..., None])[..., 0]
        except np.linalg.LinAlgError:
            delta = np.full_like(Xm, np.nan)
            for r in range(len(idx)):
                try:
                    delta[r] = np.linalg.solve(Jm[r], X[idx[r]] - Xm[r])
                except np.linalg.LinAlgError:
                    pass
        bad = ~np.all(np.isfinite(delta), axis=1)
        xi[idx] = xi[idx] + np.where(bad[:, None], 0.0, delta)
        far = np.any(np.abs(xi[idx] - (cells[idx] + 0.5)) > 4.0, axis=1)
        alive[idx[bad | far]] = False
        small = np.all(np.abs(delta) <= NEWTON_TOL, axis=1)
        conv[idx[small & ~bad & ~far]] = True
    inside = np.all((xi >= cells - SNAP) & (xi <= cells + 1 + SNAP), axis=1)
    return xi, conv & alive & inside


def snap(xi):
    r = np.round(xi)
    return np.where(np.abs(xi - r) <= SNAP, r, xi)


def find_cells(mesh, X, chunk=512, bb=None):
    """Logical coordinates (unwrapped, snapped) of points X (Q, d) in `mesh`; NaN where no cell
    contains the point (rule R17 above)."""
    X = np.asarray(X, dtype=np.float64).reshape(-1, mesh.dim)
    out = np.full(X.shape, np.nan)
    if len(X) == 0:
        return out
    cells_all, lo_all, hi_all, blocks = bb if bb is not None else cell_bboxes(mesh)
    order, starts, ends, blo, bhi = blocks
    for q0 in range(0, len(X), chunk):
        Xc = X[q0:q0 + chunk]
        # cells whose box meets the chunk's box (a pure pre-filter; flat order preserved):
        # first the blocks whose union box meets it, then their cells, re-sorted
        cmax, cmin = Xc.max(axis=0), Xc.min(axis=0)
        kb = np.nonzero(np.all((blo <= cmax) & (bhi >= cmin), axis=1))[0]
        if len(kb) == 0:
            continue
        cand = np.sort(np.concatenate([order[starts[b]:ends[b]] for b in kb]))
        keep = cand[np.all((lo_all[cand] <= cmax) & (hi_all[cand] >= cmin), axis=1)]
        cells, lo, hi = cells_all[keep], lo_all[keep], hi_all[keep]
        hit = np.ones((len(Xc), len(keep)), dtype=bool)
        for k in range(mesh.dim):
            hit &= (Xc[:, None, k] >= lo[None, :, k]) & (Xc[:, None, k] <= hi[None, :, k])
        cand = [np.nonzero(hit[q])[0] for q in range(len(Xc))]     # ascending flat cell order
        unresolved = np.ones(len(Xc), dtype=bool)
        rank = 0
        while True:
            qs = [q for q in range(len(Xc)) if unresolved[q] and rank < len(cand[q])]
            if not qs:
                break
            qs = np.array(qs)
            cs = cells[np.array([cand[q][rank] for q in qs])]
            xi, ok = _newton(mesh, Xc[qs], cs)
            for r, q in enumerate(qs):
                if ok[r]:
                    out[q0 + q] = snap(xi[r])
                    unresolved[q] = False
            rank += 1
    return out


def stencil_base(mesh, xi):
    """Interpolation base s = floor(xi) - 1, clamped (non-periodic) or left unwrapped (periodic)."""
    i0 = np.floor(xi).astype(np.int64)
    s = i0 - 1
    for k in range(mesh.dim):
        if not mesh.periodic[k]:
            s[..., k] = np.clip(s[..., k], 0, mesh.shape[k] - 4)
    return s


def shift_order(d):
    """delta in {0,+1,-1}^d ordered by sum|delta|, then lexicographically (axis 0 most
    significant) with 0 < +1 < -1."""
    rank = {0: 0, 1: 1, -1: 2}
    deltas = list(itertools.product([0, 1, -1], repeat=d))
    deltas.sort(key=lambda t: (sum(abs(v) for v in t), [rank[v] for v in t]))
    return [np.array(t, dtype=np.int64) for t in deltas]


def stencil_flat(mesh, base):
    """Flat indices (4^d,) of the stencil at unwrapped base (d,), i fastest; None if it
    leaves a non-periodic mesh."""
    offs = _stencil_offsets(mesh.dim)
    idx = base[None, :] + offs
    for k in range(mesh.dim):
        n = mesh.shape[k]
        if mesh.periodic[k]:
            idx[:, k] = np.mod(idx[:, k], n)
        elif idx[:, k].min() < 0 or idx[:, k].max() > n - 1:
            return None
    return flat_index(mesh.shape, idx)


def in_wall_body(mesh_w, X):
    """Even-odd ray test of points X (Q, 2) against the closed curve formed by the WALL face
    nodes of 2-D mesh `mesh_w` (face normal direction must be non-periodic, the other
    periodic)."""
    X = np.asarray(X, dtype=np.float64)
    inside = np.zeros(len(X), dtype=bool)
    if mesh_w.dim != 2:
        return inside
    for kap in range(2):
        for side in range(2):
            if mesh_w.face_bc[kap][side] != WALL:
                continue
            other = 1 - kap
            n_o = mesh_w.shape[other]
            j = 0 if side == 0 else mesh_w.shape[kap] - 1
            idx = np.zeros((n_o, 2), dtype=np.int64)
            idx[:, other] = np.arange(n_o)
            idx[:, kap] = j
            poly = node_coords(mesh_w, idx)
            x, y = X[:, 0], X[:, 1]
            cnt = np.zeros(len(X), dtype=bool)
            for e in range(n_o):
                x1, y1 = poly[e]
                x2, y2 = poly[(e + 1) % n_o]
                cond = (y1 > y) != (y2 > y)
                with np.errstate(divide="ignore", invalid="ignore"):
                    xint = x1 + (y - y1) * (x2 - x1) / (y2 - y1)
                cnt ^= cond & (x < xint)
            inside |= cnt
    return inside


# -------------------------------------------------------------------------------------
# the setup
# -------------------------------------------------------------------------------------
@dataclass
class Receivers:
    point: np.ndarray      # (R,) flat point index in the receiving mesh
    donor: np.ndarray      # (R,) donor mesh index
    base: np.ndarray       # (R, d) stencil base in the donor mesh (wrapped into [0, n))
    weights: np.ndarray    # (R, d, 4) per-axis Lagrange weights
    xi: np.ndarray         # (R, d) donor logical coordinates (unwrapped)


@dataclass
class OversetSetup:
    active: List[np.ndarray]        # per mesh bool, spatial shape
    positions: List[list]           # per mesh, per direction (a, b)
    receivers: List[Receivers]      # per mesh


def _face_points(mesh, bc):
    """Flat indices of the points on faces whose tag is `bc` (non-periodic directions)."""
    d = mesh.dim
    mask = np.zeros(tuple(reversed(mesh.shape)), dtype=bool)
    for k in range(d):
        if mesh.periodic[k]:
            continue
        ax = d - 1 - k
        for side in range(2):
            if mesh.face_bc[k][side] == bc:
                sl = [slice(None)] * d
                sl[ax] = 0 if side == 0 else mesh.shape[k] - 1
                mask[tuple(sl)] = True
    return np.nonzero(mask.ravel())[0]


def _flat_to_idx(shape, flat):
    idx = np.zeros((len(flat), len(shape)), dtype=np.int64)
    rem = np.asarray(flat, dtype=np.int64)
    for k in range(len(shape)):
        idx[:, k] = rem % shape[k]
        rem = rem // shape[k]
    return idx


def _points(mesh, flat):
    return mesh.xyz.reshape(mesh.dim, -1)[:, flat].T


def _priority_order(meshes, exclude):
    order = [g for g in range(len(meshes)) if g != exclude]
    order.sort(key=lambda g: (-meshes[g].priority, g))
    return order


def _global_bbox(mesh):
    X = mesh.xyz.reshape(mesh.dim, -1)
    lo, hi = X.min(axis=1), X.max(axis=1)
    g = BBOX_GROW * (hi - lo) + BBOX_ABS
    return lo - g, hi + g


def receiver_mask(mesh, positions):
    """Active points ending a segment next to a hole or an OVERSET face (any direction)."""
    d = mesh.dim
    shp = tuple(reversed(mesh.shape))
    recv = np.zeros(shp, dtype=bool)
    for k in range(d):
        a, b = positions[k]
        ax = d - 1 - k
        n = mesh.shape[k]
        idx = np.arange(n).reshape([n if i == ax else 1 for i in range(d)])
        for side, pos in ((0, a), (1, b)):
            end = pos == 0
            at_face = (idx == 0) if side == 0 else (idx == n - 1)
            if mesh.periodic[k]:
                recv |= end                                  # a periodic end is always a hole
            else:
                across_hole = end & ~at_face
                across_overset = end & at_face & (mesh.face_bc[k][side] == OVERSET)
                recv |= across_hole | across_overset
    return recv


def build_overset(meshes) -> OversetSetup:
    G = len(meshes)
    bbs = [cell_bboxes(m) for m in meshes]
    gbb = [_global_bbox(m) for m in meshes]
    inside = [np.zeros(tuple(reversed(m.shape)), dtype=bool) for m in meshes]
    # 1. A-points inside higher-priority meshes or inside wall bodies
    for A in range(G):
        XA = meshes[A].xyz.reshape(meshes[A].dim, -1).T
        flatin = inside[A].ravel()
        for B in range(G):
            if B == A:
                continue
            if meshes[B].priority > meshes[A].priority:
                lo, hi = gbb[B]
                sel = np.nonzero(np.all((XA >= lo) & (XA <= hi), axis=1))[0]
                xi = find_cells(meshes[B], XA[sel], bb=bbs[B])
                flatin[sel[np.all(np.isfinite(xi), axis=1)]] = True
            flatin |= in_wall_body(meshes[B], XA)
        inside[A] = flatin.reshape(inside[A].shape)
    # 2. protect the donor stencils of overset-face points
    protected = [np.zeros_like(x) for x in inside]
    for B in range(G):
        fpts = _face_points(meshes[B], OVERSET)
        if len(fpts) == 0:
            continue
        Xf = _points(meshes[B], fpts)
        todo = np.ones(len(fpts), dtype=bool)
        for A in _priority_order(meshes, B):
            sel = np.nonzero(todo)[0]
            if len(sel) == 0:
                break
            xi = find_cells(meshes[A], Xf[sel], bb=bbs[A])
            ok = np.all(np.isfinite(xi), axis=1)
            pflat = protected[A].ravel()
            for r in np.nonzero(ok)[0]:
                base = stencil_base(meshes[A], xi[r])
                st = stencil_flat(meshes[A], base)
                pflat[st] = True
            protected[A] = pflat.reshape(protected[A].shape)
            todo[sel[ok]] = False
    # 3. blanking
    active = [~(inside[g] & ~protected[g]) for g in range(G)]
    # 4. segments, receivers, donors
    positions = []
    for g, m in enumerate(meshes):
        pos = [sbp.segment_positions(active[g], m.dim - 1 - k, m.periodic[k])
               for k in range(m.dim)]
        for k in range(m.dim):
            if sbp.check_segments(*pos[k]) < sbp.MIN_SEGMENT:
                raise SegmentTooShort(f"mesh {g} direction {k}: segment shorter than "
                                      f"{sbp.MIN_SEGMENT}")
        positions.append(pos)
    receivers = []
    for g, m in enumerate(meshes):
        pts = np.nonzero(receiver_mask(m, positions[g]).ravel())[0]
        X = _points(m, pts)
        R = len(pts)
        donor = np.full(R, -1, dtype=np.int64)
        base = np.zeros((R, m.dim), dtype=np.int64)
        wts = np.zeros((R, m.dim, 4))
        xis = np.zeros((R, m.dim))
        todo = np.ones(R, dtype=bool)
        for A in _priority_order(meshes, g):
            sel = np.nonzero(todo)[0]
            if len(sel) == 0:
                break
            xi = find_cells(meshes[A], X[sel], bb=bbs[A])
            act = active[A].ravel()
            for r, q in enumerate(sel):
                if not np.all(np.isfinite(xi[r])):
                    continue
                s0 = stencil_base(meshes[A], xi[r])
                for delta in shift_order(m.dim):
                    s = s0 + delta
                    st = stencil_flat(meshes[A], s)
                    if st is None or not act[st].all():
                        continue
                    donor[q] = A
                    wrapped = s.copy()
                    for k in range(m.dim):
                        if meshes[A].periodic[k]:
                            wrapped[k] = s[k] % meshes[A].shape[k]
                    base[q] = wrapped
                    wts[q] = lagrange_weights(xi[r] - s)
                    xis[q] = xi[r]
                    todo[q] = False
                    break
        if todo.any():
            bad = pts[todo][:4]
            raise OrphanReceiver(f"mesh {g}: {int(todo.sum())} receivers without donor, e.g. "
                                 f"points {bad.tolist()} at {_points(m, bad).tolist()}")
        receivers.append(Receivers(pts, donor, base, wts, xis))
    return OversetSetup(active, positions, receivers)
