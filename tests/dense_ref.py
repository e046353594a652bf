"""Dense brute-force reference of the coupled 2-D SBP-SAT right-hand side (test infrastructure).

Independent of oracle/rhs.py: every operator is an explicit matrix assembled here from the
paper's definitions, and the RHS is a chain of dense matrix-vector products --
  * D_kappa: the diagonal-norm 2-4 first-derivative operator (coefficients of
    App. A typed below) placed block by block on every maximal run of active points of every
    grid line (reading R2), cyclic interior stencil on hole-free periodic lines;
  * metrics: x_xi = D_xi x etc., M_xi = (y_eta, -x_eta), M_eta = (-y_xi, x_xi),
    J^-1 = x_xi y_eta - x_eta y_xi (reading R3);
  * gradients d_i phi = J sum_kappa M_kappa,i D_kappa phi, tau, heat flux (R11), fluxes
    F_i = F^I_i - F^V_i, Fhat_kappa = sum_i M_kappa,i F_i, R = -J sum_kappa D_kappa Fhat_kappa
    (eq:int);
  * SAT (readings R14-R19): at each run end (kappa, side) facing a hole, an
    overset face or a physical face, with K^side built by a NUMERICAL eigendecomposition of the
    analytic flux Jacobian A(n) (the oracle uses complex-step + Sylvester, the GPU the analytic
    eigenvectors) and qhat from an explicit interpolation matrix whose rows are tensor Lagrange
    weights recomputed here from the donor logical coordinates.
Inputs taken from the oracle's overset setup: the active masks and, per receiver, the donor
mesh, stencil base and donor logical coordinates (the hole cutting / donor search is pinned
separately by brute force in test_oracle_overset.py); the receiver SET is recomputed here
from the run ends and must equal the oracle's.  2-D, meshes without coordinate jumps across
periodic seams (closed O-grids, non-periodic Cartesian meshes).
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np

OVERSET, FARFIELD, WALL, PERIODIC = 0, 1, 2, 3

# App. A: left closure rows of the 2-4 operator (columns 0..5) and the interior stencil
_LEFT = [[Fr(-24, 17), Fr(59, 34), Fr(-4, 17), Fr(-3, 34), 0, 0],
         [Fr(-1, 2), 0, Fr(1, 2), 0, 0, 0],
         [Fr(4, 43), Fr(-59, 86), 0, Fr(59, 86), Fr(-4, 43), 0],
         [Fr(3, 98), 0, Fr(-59, 98), 0, Fr(32, 49), Fr(-4, 49)]]
_INT = {-2: Fr(1, 12), -1: Fr(-2, 3), 1: Fr(2, 3), 2: Fr(-1, 12)}
P0 = 17.0 / 48.0


def sbp_matrix(L):
    """Dense D1 (L x L) of one segment: closure rows at both ends, D[L-1-r][L-1-c] = -D[r][c]."""
    D = np.zeros((L, L))
    for r in range(L):
        for o, c in _INT.items():
            if 0 <= r + o < L:
                D[r, r + o] = float(c)
    for r in range(4):
        D[r, :] = 0.0
        D[L - 1 - r, :] = 0.0
    for r in range(4):
        for c in range(6):
            D[r, c] = float(_LEFT[r][c])
            D[L - 1 - r, L - 1 - c] = -float(_LEFT[r][c])
    return D


def cyclic_matrix(n):
    D = np.zeros((n, n))
    for r in range(n):
        for o, c in _INT.items():
            D[r, (r + o) % n] += float(c)
    return D


def _lines(shape, k):
    """Flat index arrays of every grid line along direction k (index order, i fastest)."""
    n0, n1 = shape
    if k == 0:
        return [np.arange(n0) + n0 * j for j in range(n1)]
    return [i + n0 * np.arange(n1) for i in range(n0)]


def runs(active_line, periodic):
    """Maximal runs of active points along one line, as lists of positions in line order
    (a run may wrap across the seam of a periodic line); None = hole-free periodic line."""
    n = len(active_line)
    if periodic and active_line.all():
        return None
    start = 0
    if periodic:
        start = int(np.nonzero(~active_line)[0][0])          # begin scanning at a hole
    out, cur = [], []
    for t in range(n):
        pos = (start + t) % n
        if active_line[pos]:
            cur.append(pos)
        elif cur:
            out.append(cur)
            cur = []
    if cur:
        out.append(cur)
    return out


def derivative_matrix(mesh, active, k):
    """Dense D_kappa (N x N) of one mesh and the run ends: ends[(p, side)] for side +1 (run
    start) / -1 (run end), each with the flag 'at a physical face'."""
    N = mesh.npts
    D = np.zeros((N, N))
    ends = {}
    act = active.ravel()
    for line in _lines(mesh.shape, k):
        rs = runs(act[line], mesh.periodic[k])
        if rs is None:
            D[np.ix_(line, line)] = cyclic_matrix(len(line))
            continue
        for run in rs:
            idx = line[np.array(run)]
            D[np.ix_(idx, idx)] = sbp_matrix(len(run))
            n = len(line)
            ends[(int(idx[0]), +1)] = (not mesh.periodic[k]) and run[0] == 0
            ends[(int(idx[-1]), -1)] = (not mesh.periodic[k]) and run[-1] == n - 1
    return D, ends


def lagrange(t):
    return np.array([np.prod([(t - b) / (a - b) for b in range(4) if b != a]) for a in range(4)])


def flux_jacobian(q, n, gamma):
    """Analytic A(n) = sum_i n_i dF^I_i/dq of the 2-D Euler flux."""
    rho, m1, m2, E = q
    u, v = m1 / rho, m2 / rho
    g1 = gamma - 1.0
    un = u * n[0] + v * n[1]
    ke = 0.5 * (u * u + v * v)
    H = (E + g1 * (E - rho * ke)) / rho
    return np.array([
        [0.0, n[0], n[1], 0.0],
        [g1 * ke * n[0] - u * un, un + u * n[0] - g1 * u * n[0], u * n[1] - g1 * v * n[0], g1 * n[0]],
        [g1 * ke * n[1] - v * un, v * n[0] - g1 * u * n[1], un + v * n[1] - g1 * v * n[1], g1 * n[1]],
        [(g1 * ke - H) * un, H * n[0] - g1 * u * un, H * n[1] - g1 * v * un, gamma * un]])


def k_side(q, n, side, gamma):
    """K^side = T diag(max(side lambda, 0)) T^-1 by numerical linear algebra: LAPACK eig for the
    two simple eigenvalues, and for the double one (the closest pair of computed eigenvalues)
    an SVD null-space basis of A - lambda_0 I (eig alone may return a near-dependent pair of
    eigenvectors there)."""
    A = flux_jacobian(q, n, gamma)
    lam, V = np.linalg.eig(A)
    lam = lam.real
    pairs = [(abs(lam[a] - lam[b]), a, b) for a in range(4) for b in range(a + 1, 4)]
    _, a, b = min(pairs)
    lam0 = 0.5 * (lam[a] + lam[b])
    simple = [k for k in range(4) if k not in (a, b)]
    _, _, Vt = np.linalg.svd(A - lam0 * np.eye(4))
    T = np.column_stack([V[:, simple[0]].real, V[:, simple[1]].real, Vt[-1], Vt[-2]])
    ev = np.array([lam[simple[0]], lam[simple[1]], lam0, lam0])
    return (T * np.maximum(side * ev, 0.0)[None, :]) @ np.linalg.inv(T)


class DenseRHS:
    def __init__(self, problem, ov):
        self.p = problem
        self.G = len(problem.meshes)
        self.D, self.ends, self.J, self.M = [], [], [], []
        for g, m in enumerate(problem.meshes):
            assert m.dim == 2
            for k in range(2):
                assert not any(m.period[k]), "coordinate jumps across seams are not modelled"
            Dx, ex = derivative_matrix(m, ov.active[g], 0)
            Dy, ey = derivative_matrix(m, ov.active[g], 1)
            x, y = m.xyz[0].ravel(), m.xyz[1].ravel()
            xx, xy, yx, yy = Dx @ x, Dy @ x, Dx @ y, Dy @ y        # x_xi, x_eta, y_xi, y_eta
            jinv = xx * yy - xy * yx
            act = ov.active[g].ravel()
            J = np.where(act, 1.0 / np.where(act, jinv, 1.0), 0.0)
            self.D.append((Dx, Dy))
            self.ends.append((ex, ey))
            self.J.append(J)
            self.M.append(((yy, -xy), (-yx, xx)))                   # M[kappa][i]
        self.active = [a.ravel() for a in ov.active]
        # explicit interpolation matrices: receiver (g, point) -> (donor mesh, row)
        self.interp = []
        for g in range(self.G):
            rc = ov.receivers[g]
            rows = {}
            for r, pnt in enumerate(rc.point):
                dm = problem.meshes[rc.donor[r]]
                row = np.zeros(dm.npts)
                w0 = lagrange(rc.xi[r, 0] - self._unwrap(rc.base[r, 0], rc.xi[r, 0], dm, 0))
                w1 = lagrange(rc.xi[r, 1] - self._unwrap(rc.base[r, 1], rc.xi[r, 1], dm, 1))
                for b in range(4):
                    for a in range(4):
                        i = (rc.base[r, 0] + a) % dm.shape[0]
                        j = (rc.base[r, 1] + b) % dm.shape[1]
                        row[i + dm.shape[0] * j] += w0[a] * w1[b]
                rows[int(pnt)] = (int(rc.donor[r]), row)
            self.interp.append(rows)

    @staticmethod
    def _unwrap(base, xi, mesh, k):
        # logical coordinate and (wrapped) base may sit on opposite sides of a periodic seam
        if mesh.periodic[k] and xi - base > 3.5:
            return base + mesh.shape[k]
        if mesh.periodic[k] and xi - base < -0.5:
            return base - mesh.shape[k]
        return base

    def receiver_points(self, g):
        """Run ends facing a hole or an OVERSET face (recomputed from the runs)."""
        m = self.p.meshes[g]
        pts = set()
        for k in range(2):
            for (pnt, side), at_face in self.ends[g][k].items():
                bc = m.face_bc[k][0 if side > 0 else 1]
                if not at_face or bc == OVERSET:
                    pts.add(pnt)
        return sorted(pts)

    def _prims(self, q):
        gam = self.p.gamma
        rho = q[0]
        u, v = q[1] / rho, q[2] / rho
        p = (gam - 1.0) * (q[3] - 0.5 * rho * (u * u + v * v))
        return rho, u, v, p, gam * p / rho

    def viscous_fluxes(self, g, q):
        """Cartesian F^V_i (4, N) for i = 0, 1 (zeros if inviscid)."""
        N = q.shape[1]
        if not self.p.viscous:
            return [np.zeros((4, N)), np.zeros((4, N))]
        Dx, Dy = self.D[g]
        J, M = self.J[g], self.M[g]
        rho, u, v, p, T = self._prims(q)
        grad = {}
        for name, f in (("u", u), ("v", v), ("T", T)):
            dk = (Dx @ f, Dy @ f)
            grad[name] = [J * (M[0][i] * dk[0] + M[1][i] * dk[1]) for i in range(2)]
        mu_re = 1.0 / self.p.Re
        kT = 1.0 / (self.p.Re * self.p.Pr * (self.p.gamma - 1.0))
        ux, uy = grad["u"]
        vx, vy = grad["v"]
        div = ux + vy
        txx = mu_re * (2 * ux - 2.0 / 3.0 * div)
        tyy = mu_re * (2 * vy - 2.0 / 3.0 * div)
        txy = mu_re * (uy + vx)
        fx = np.stack([np.zeros(N), txx, txy, u * txx + v * txy + kT * grad["T"][0]])
        fy = np.stack([np.zeros(N), txy, tyy, u * txy + v * tyy + kT * grad["T"][1]])
        return [fx, fy]

    def rhs(self, states):
        P = self.p
        qs = [s.reshape(4, -1) for s in states]
        FV = [self.viscous_fluxes(g, qs[g]) for g in range(self.G)]
        out = []
        for g in range(self.G):
            m = P.meshes[g]
            q = qs[g]
            Dx, Dy = self.D[g]
            J, M = self.J[g], self.M[g]
            rho, u, v, p, T = self._prims(q)
            E = q[3]
            FI = [np.stack([rho * u, rho * u * u + p, rho * u * v, (E + p) * u]),
                  np.stack([rho * v, rho * u * v, rho * v * v + p, (E + p) * v])]
            F = [FI[i] - FV[g][i] for i in range(2)]
            Fh = [M[k][0][None] * F[0] + M[k][1][None] * F[1] for k in range(2)]
            R = -J[None] * ((Dx @ Fh[0].T).T + (Dy @ Fh[1].T).T)
            R[:, ~self.active[g]] = 0.0
            for k in range(2):
                for (pnt, side), at_face in self.ends[g][k].items():
                    typ = m.face_bc[k][0 if side > 0 else 1] if at_face else OVERSET
                    nvec = np.array([J[pnt] * M[k][0][pnt], J[pnt] * M[k][1][pnt]])
                    qp = q[:, pnt]
                    if typ == OVERSET:
                        dmesh, row = self.interp[g][pnt]
                        qh = qs[dmesh] @ row
                    elif typ == FARFIELD:
                        qh = np.asarray(P.q_inf[:4], dtype=np.float64)
                    elif typ == WALL:
                        qh = np.array([qp[0], 0.0, 0.0, qp[0] * P.wall_T / (P.gamma * (P.gamma - 1.0))])
                    else:
                        raise AssertionError("periodic faces have no run ends")
                    dq = qp - qh
                    pen = 0.5 * k_side(qp, nvec, side, P.gamma) @ dq
                    if P.viscous:
                        pen = pen + (nvec @ nvec) / (2.0 * P.Re) * dq
                    sat = -pen / P0
                    if P.viscous and typ != WALL:
                        fvk = nvec[0] * FV[g][0][:, pnt] + nvec[1] * FV[g][1][:, pnt]
                        if typ == OVERSET:
                            dmesh, row = self.interp[g][pnt]
                            fvh = nvec[0] * (FV[dmesh][0] @ row) + nvec[1] * (FV[dmesh][1] @ row)
                        else:
                            fvh = 0.0
                        sat = sat + 0.5 * side * (fvk - fvh) / P0
                    R[:, pnt] += sat
            out.append(R.reshape(states[g].shape))
        return out
