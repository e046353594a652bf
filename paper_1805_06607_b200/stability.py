"""Step-matrix stability laboratory on the GPU path.

PAPER.md §5.1: phi_{n+1} ~ G_eps phi_n (eq:sm); column j of G_eps is
(step(phi + eps e_j) - step(phi)) / eps (eq:sm_form), eps = 1e-7, history entries included in
phi; stable iff rho(G_eps) <= 1.  Every application of the map is one mrab_step of the CUDA
path (libmrab.so) from an integrator vector written into the context with mrab_set_state /
mrab_set_history; the host only forms differences and solves the eigenproblem (dense for the
full matrix, ARPACK Arnoldi on the matrix-free operator for large vectors -- the paper uses
SLEPc's Krylov-Schur, tolerance 1e-12).

Integrator vector (reading R-SM): per mesh g, its state then its m-1 committed RHS
history entries, oldest first, all dense [nc][n...] fp64.
"""
from __future__ import annotations

import numpy as np

from . import mrab

EPS = 1e-7


class StepMap:
    """phi -> phi' = one MRAB macro step on the GPU.  The context must be past its bootstrap
    (m-1 macro steps); the map is time-independent because the RHS is autonomous."""

    def __init__(self, ctx: "mrab.Context"):
        self.ctx = ctx
        P = ctx.plan
        self.m = P.history_m
        self.shapes = [(P.nc,) + tuple(reversed(P.shapes[g])) for g in range(P.n_meshes)]
        self.sizes = [int(np.prod(s)) for s in self.shapes]
        self.dim = sum(self.sizes) * self.m

    def read(self):
        """Current integrator vector of the context."""
        parts = []
        for g, shp in enumerate(self.shapes):
            parts.append(self.ctx.get_state(g)[0].ravel())
            for k in range(self.m - 1):
                parts.append(self.ctx.get_history(g, k).ravel())
        return np.concatenate(parts)

    def write(self, phi):
        o = 0
        for g, (shp, n) in enumerate(zip(self.shapes, self.sizes)):
            self.ctx.set_state(g, np.ascontiguousarray(phi[o:o + n].reshape(shp)))
            o += n
            for k in range(self.m - 1):
                self.ctx.set_history(g, k, np.ascontiguousarray(phi[o:o + n].reshape(shp)))
                o += n
        assert o == phi.size

    def __call__(self, phi):
        self.write(phi)
        self.ctx.step(1)
        return self.read()

    # ---- device-resident variant: the integrator vector stays on the GPU (torch tensors), the
    # accessors copy device to device, so forming a column costs no host round trip
    def read_device(self, out=None):
        import torch
        if out is None:
            out = torch.empty(self.dim, dtype=torch.float64, device="cuda")
        o = 0
        for g, n in enumerate(self.sizes):
            self.ctx.get_state(g, out=out[o:o + n])
            o += n
            for k in range(self.m - 1):
                self.ctx.get_history(g, k, out=out[o:o + n])
                o += n
        return out

    def write_device(self, phi):
        o = 0
        for g, n in enumerate(self.sizes):
            self.ctx.set_state(g, phi[o:o + n])
            o += n
            for k in range(self.m - 1):
                self.ctx.set_history(g, k, phi[o:o + n])
                o += n

    def apply_device(self, phi, out=None):
        self.write_device(phi)
        self.ctx.step(1)
        return self.read_device(out)


def step_matrix_device(smap: StepMap, phi0, eps=EPS, cols=None):
    """G_eps (eq:sm_form) with every vector resident on the GPU: phi0 is perturbed on the
    device, written into the context by device-to-device copies, stepped, read back on the
    device and differenced there; the matrix is returned as a CUDA tensor (columns `cols`)."""
    import torch
    phi0 = torch.as_tensor(phi0, dtype=torch.float64, device="cuda")
    base = smap.apply_device(phi0).clone()
    cols = list(range(phi0.numel())) if cols is None else list(cols)
    G = torch.empty((base.numel(), len(cols)), dtype=torch.float64, device="cuda")
    ph = phi0.clone()
    buf = torch.empty_like(base)
    for c, j in enumerate(cols):
        ph[j] += eps
        smap.apply_device(ph, out=buf)
        G[:, c] = (buf - base) / eps
        ph[j] = phi0[j]
    return G


class RKMap:
    """phi -> phi' = one step of size h of the reference Runge-Kutta integrator (classical RK4
    by default; P:861-878 normalises the stability tables by its maximum stable step) on the
    GPU (mrab_rk_step).  The integrator vector is the states only."""

    def __init__(self, ctx: "mrab.Context", h, order=4):
        self.ctx, self.h, self.order = ctx, float(h), int(order)
        P = ctx.plan
        self.shapes = [(P.nc,) + tuple(reversed(P.shapes[g])) for g in range(P.n_meshes)]
        self.sizes = [int(np.prod(s)) for s in self.shapes]
        self.dim = sum(self.sizes)

    def read(self):
        return np.concatenate([self.ctx.get_state(g)[0].ravel() for g in range(len(self.shapes))])

    def write(self, phi):
        o = 0
        for g, (shp, n) in enumerate(zip(self.shapes, self.sizes)):
            self.ctx.set_state(g, np.ascontiguousarray(phi[o:o + n].reshape(shp)))
            o += n

    def __call__(self, phi):
        self.write(phi)
        self.ctx.rk_step(self.h, 1, self.order)
        return self.read()


def spectral_radius_arnoldi(smap, phi0, k=80, restarts=6, eps=EPS, seed=0, res_tol=1e-6):
    """Largest modulus among the CONVERGED eigenvalues of G_eps, by explicitly restarted Arnoldi
    on the matrix-free operator v -> (step(phi0 + eps v/|v|) - step(phi0)) |v| / eps: k steps
    build an orthonormal Krylov basis (Gram-Schmidt twice); a Ritz pair (theta, V y) counts as
    converged when its residual |h_{k+1,k}| |y_k| <= res_tol |theta| (Ritz values of a
    non-normal step matrix that have not converged can lie outside its spectrum, so they are
    not used); the iteration restarts from the sum of the leading Ritz vectors until the leading
    pair has converged.  A plain stand-in for the Krylov-Schur solver the paper uses.
    Non-finite steps (blow-up) return inf; no converged pair returns 0.  Returns (rho, matvecs)."""
    base = smap(phi0)
    if not np.all(np.isfinite(base)):
        return float("inf"), 1
    n = phi0.size
    v = np.random.default_rng(seed).standard_normal(n)
    nmv, best = 1, 0.0
    for _ in range(restarts):
        V = np.zeros((k + 1, n))
        Hm = np.zeros((k + 1, k))
        V[0] = v / np.linalg.norm(v)
        kk = k
        for j in range(k):
            w = (smap(phi0 + eps * V[j]) - base) / eps
            nmv += 1
            if not np.all(np.isfinite(w)):
                return float("inf"), nmv
            for _pass in range(2):
                c = V[:j + 1] @ w
                w = w - c @ V[:j + 1]
                Hm[:j + 1, j] += c
            Hm[j + 1, j] = np.linalg.norm(w)
            if Hm[j + 1, j] < 1e-14:
                kk = j + 1
                break
            V[j + 1] = w / Hm[j + 1, j]
        ev, Y = np.linalg.eig(Hm[:kk, :kk])
        res = np.abs(Hm[kk, kk - 1]) * np.abs(Y[kk - 1, :]) if kk == k else np.zeros(kk)
        order = np.argsort(-np.abs(ev))
        conv = [i for i in order if res[i] <= res_tol * max(abs(ev[i]), 1e-300)]
        if conv:
            best = max(best, float(abs(ev[conv[0]])))
        if res[order[0]] <= res_tol * abs(ev[order[0]]):
            break                                     # the leading pair itself has converged
        lead = order[:min(4, kk)]
        v = np.real(Y[:, lead].sum(axis=1)) @ V[:kk]
        if np.linalg.norm(v) < 1e-12:
            v = np.imag(Y[:, lead].sum(axis=1)) @ V[:kk]
    return best, nmv


def growth_rate(smap, phi0, iters=300, eps=EPS, seed=0):
    """Asymptotic growth factor per step of a perturbation under the linearised map:
    exp(mean log-norm slope over the second half of `iters` renormalised power iterations).
    It approaches rho(G_eps) from the dominant mode and, unlike unconverged Ritz values, does
    not overshoot once the transient has decayed.  Blow-up returns inf."""
    base = smap(phi0)
    if not np.all(np.isfinite(base)):
        return float("inf")
    v = np.random.default_rng(seed).standard_normal(phi0.size)
    v /= np.linalg.norm(v)
    logs = []
    for _ in range(iters):
        w = (smap(phi0 + eps * v) - base) / eps
        nw = float(np.linalg.norm(w))
        if not np.isfinite(nw) or nw == 0.0:
            return float("inf") if not np.isfinite(nw) else 0.0
        logs.append(np.log(nw))
        v = w / nw
    half = iters // 2
    return float(np.exp(np.mean(logs[half:])))


def step_matrix(smap: StepMap, phi0, eps=EPS, cols=None):
    """G_eps (eq:sm_form), all columns or the listed ones."""
    base = smap(phi0)
    cols = range(phi0.size) if cols is None else cols
    G = np.empty((base.size, len(cols)))
    for c, j in enumerate(cols):
        ph = phi0.copy()
        ph[j] += eps
        G[:, c] = (smap(ph) - base) / eps
    return G


def spectral_radius(G):
    return float(np.max(np.abs(np.linalg.eigvals(G))))


def spectral_radius_krylov(smap: StepMap, phi0, eps=EPS, tol=1e-12, maxiter=None, seed=0):
    """rho(G_eps) from the matrix-free operator v -> (step(phi0 + eps v/|v|) - step(phi0))
    |v| / eps (ARPACK, largest magnitude)."""
    from scipy.sparse.linalg import LinearOperator, eigs
    base = smap(phi0)

    def mv(v):
        v = np.real(np.asarray(v, dtype=np.complex128)).ravel()
        nv = np.linalg.norm(v)
        if nv == 0.0:
            return np.zeros_like(v)
        return (smap(phi0 + (eps / nv) * v) - base) * (nv / eps)

    op = LinearOperator((phi0.size, phi0.size), matvec=mv, dtype=np.float64)
    v0 = np.random.default_rng(seed).standard_normal(phi0.size)
    vals = eigs(op, k=1, which="LM", tol=tol, maxiter=maxiter, v0=v0,
                return_eigenvectors=False)
    return float(np.max(np.abs(vals)))


def power_estimate(smap: StepMap, phi0, iters=30, eps=EPS, seed=0):
    """|G^k v| / |G^(k-1) v| after `iters` matrix-free power iterations from a seeded
    vector (a bounded-cost lower estimate of rho(G_eps))."""
    base = smap(phi0)
    v = np.random.default_rng(seed).standard_normal(phi0.size)
    v /= np.linalg.norm(v)
    est = 0.0
    for _ in range(iters):
        w = (smap(phi0 + eps * v) - base) / eps
        est = float(np.linalg.norm(w))
        v = w / est
    return est


def max_stable(rho_of, lo, hi, tol=1e-4, one=1.0):
    """Largest x in [lo, hi] with rho_of(x) <= one by bisection to tol.  `one` > 1
    absorbs the finite-difference noise of eq:sm_form on neutral modes (DESIGN.md R-SM)."""
    if rho_of(hi) <= one:
        return hi
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if rho_of(mid) <= one:
            lo = mid
        else:
            hi = mid
    return lo
