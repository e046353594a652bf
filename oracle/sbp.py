"""Diagonal-norm SBP 2-4 first-derivative operator on segments (ORACLE, test infrastructure).

PAPER.md P:205-208 (§2.1): "we use the third-order SBP operator given in
[mattsson2004stable]"; P:797-799 ("fourth-order SBP operator"), P:1526-1528 ("SBP 4-2",
"two applications of the first-derivative operator").  Reading R9: these
are ONE operator, the diagonal-norm 2-4 operator (interior 4th order, boundary 2nd order).
The paper prints no coefficients; the ones below are the unique diagonal-norm 2-4 set
(SURVEY.md App. A).  They are pinned in tests/test_oracle_sbp.py by the SBP property
H D + D^T H = diag(-1, 0, ..., 0, 1) in exact rationals, by polynomial exactness
(boundary rows degree 2, interior degree 4) and by the periodic symbol maximum
1.3722 of P:800-802.

Index space: unit spacing.  Along every grid line in each direction, every maximal run of
active points (a "segment", reading R2 of DESIGN.md) carries its own copy of the operator:
left closure rows at its start, mirrored right closure rows at its end, interior stencil
elsewhere.  A periodic line without holes uses the cyclic interior stencil.
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np

# H = diag(17/48, 59/48, 43/48, 49/48, 1, ..., 1, 49/48, 43/48, 59/48, 17/48)
H_BOUNDARY = (Fr(17, 48), Fr(59, 48), Fr(43, 48), Fr(49, 48))

# left closure rows r = 0..3 as {column: coefficient}
LEFT_ROWS = (
    {0: Fr(-24, 17), 1: Fr(59, 34), 2: Fr(-4, 17), 3: Fr(-3, 34)},
    {0: Fr(-1, 2), 2: Fr(1, 2)},
    {0: Fr(4, 43), 1: Fr(-59, 86), 3: Fr(59, 86), 4: Fr(-4, 43)},
    {0: Fr(3, 98), 2: Fr(-59, 98), 4: Fr(32, 49), 5: Fr(-4, 49)},
)
# interior row as {offset: coefficient}
INTERIOR = {-2: Fr(1, 12), -1: Fr(-2, 3), 1: Fr(2, 3), 2: Fr(-1, 12)}

NCLOSE = 4            # closure rows per end
MIN_SEGMENT = 8       # shortest segment on which left and right closures do not overlap
FAR = 1 << 30         # "distance to segment end" on a hole-free periodic line


def row_stencil(a: int, b: int):
    """{offset: Fraction} of the D1 row for a point at distance a from its segment start and
    b from its segment end (offsets relative to the point)."""
    if a < NCLOSE:
        return {c - a: v for c, v in LEFT_ROWS[a].items()}
    if b < NCLOSE:
        # D[N-1-r][N-1-c] = -D[r][c]  ->  offset -(c - r), coefficient -v
        return {-(c - b): -v for c, v in LEFT_ROWS[b].items()}
    return dict(INTERIOR)


def norm_weight(a: int, b: int) -> Fr:
    if a < NCLOSE:
        return H_BOUNDARY[a]
    if b < NCLOSE:
        return H_BOUNDARY[b]
    return Fr(1)


def d1_matrix(n: int, periodic: bool = False):
    """Dense D1 (list of lists of Fractions) on one segment of n points (pins only)."""
    D = [[Fr(0)] * n for _ in range(n)]
    for r in range(n):
        a, b = (FAR, FAR) if periodic else (r, n - 1 - r)
        for off, v in row_stencil(a, b).items():
            c = r + off
            if periodic:
                c %= n
            D[r][c] += v
    return D


def h_matrix(n: int):
    return [norm_weight(r, n - 1 - r) for r in range(n)]


def segment_positions(active: np.ndarray, axis: int, periodic: bool):
    """Distance of every point to the start (a) and to the end (b) of its segment along
    `axis`.  Holes get -1; points on a hole-free periodic line get FAR.  Plain loops over the
    line index (vectorised over the other axes)."""
    act = np.moveaxis(np.asarray(active, dtype=bool), axis, -1)
    n = act.shape[-1]
    a = np.full(act.shape, -1, dtype=np.int64)
    b = np.full(act.shape, -1, dtype=np.int64)
    if periodic:
        carry = np.full(act.shape[:-1], FAR, dtype=np.int64)
        for it in range(2 * n):
            i = it % n
            carry = np.where(act[..., i], np.minimum(carry + 1, FAR), -1)
            if it >= n:
                a[..., i] = carry
        carry = np.full(act.shape[:-1], FAR, dtype=np.int64)
        for it in range(2 * n):
            i = (n - 1) - (it % n)
            carry = np.where(act[..., i], np.minimum(carry + 1, FAR), -1)
            if it >= n:
                b[..., i] = carry
    else:
        carry = np.full(act.shape[:-1], -1, dtype=np.int64)
        for i in range(n):
            carry = np.where(act[..., i], carry + 1, -1)
            a[..., i] = carry
        carry = np.full(act.shape[:-1], -1, dtype=np.int64)
        for i in range(n - 1, -1, -1):
            carry = np.where(act[..., i], carry + 1, -1)
            b[..., i] = carry
    return np.moveaxis(a, -1, axis), np.moveaxis(b, -1, axis)


def check_segments(a, b):
    """Segment lengths a+b+1 of active points; returns the shortest (FAR if none closed)."""
    act = a >= 0
    if not act.any():
        return FAR
    L = np.where(act & (a < FAR) & (b < FAR), a + b + 1, FAR)
    return int(L.min())


def _row_classes():
    """(mask-builder, stencil) pairs: left rows 0..3, right rows 0..3, interior."""
    out = []
    for r in range(NCLOSE):
        out.append(("L", r, row_stencil(r, FAR)))
    for r in range(NCLOSE):
        out.append(("R", r, row_stencil(FAR, r)))
    out.append(("I", None, dict(INTERIOR)))
    return out


ROW_CLASSES = _row_classes()


def _shift(f, off, axis):
    """g[i] = f[(i + off) mod n] along axis, plus the wrap count floor((i+off)/n)."""
    n = f.shape[axis]
    g = np.roll(f, -off, axis=axis)
    idx = np.arange(n) + off
    wrap = np.floor_divide(idx, n)
    shape = [1] * f.ndim
    shape[axis] = n
    return g, wrap.reshape(shape)


def d1(f: np.ndarray, axis: int, a: np.ndarray, b: np.ndarray, jump: float = 0.0,
       factor: np.ndarray | None = None):
    """(D1 f) along `axis` with the segment positions (a, b) of that axis.

    `f` has the spatial shape of the mesh.  `jump` is the increment of f across a periodic
    seam (f(i+n) = f(i) + jump; used for coordinates).  If `factor` is given the operator is
    applied to the product jump-unwrapped(f) * factor with `factor` seam-periodic (used by
    the conservative metric forms).  Holes (a < 0) get 0.
    """
    out = np.zeros(np.broadcast_shapes(f.shape, a.shape), dtype=np.float64)
    masks = {}
    for kind, r, st in ROW_CLASSES:
        if kind == "L":
            m = a == r
        elif kind == "R":
            m = (b == r) & (a >= NCLOSE)
        else:
            m = (a >= NCLOSE) & (b >= NCLOSE)
        masks[(kind, r)] = (m, st)
    for off in sorted({o for _, _, st in ROW_CLASSES for o in st}):
        g, wrap = _shift(f, off, axis)
        if jump != 0.0:
            g = g + wrap * jump
        if factor is not None:
            g = g * _shift(factor, off, axis)[0]
        for (kind, r), (m, st) in masks.items():
            if off in st:
                out[m] += float(st[off]) * g[m]
    return out
