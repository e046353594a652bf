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
