"""RK bootstrap and N-rate fastest-first MRAB without re-extrapolation (ORACLE, test
infrastructure).

PAPER.md §3.1: AB step y(t_{i+1}) = y(t_i) + sum_k alpha_k F_k (eq:ab_general),
bootstrapped by RK3 [heun1900neue] for third-order and RK4 for fourth-order schemes.
§3.3 Steps 1-7: fastest-first, no re-extrapolation; a slow component is marched
to intermediate times by integrating its extrapolant partially from the state at the start
of its own step (Step 5 integrates from s(t_i), reading R7).  Readings:
R5 Heun RK3 c = (0, 1/3, 2/3), a21 = 1/3, a32 = 2/3, b = (1/4, 0, 3/4), used for n <= 3;
classical RK4 for n = 4.  R6 bootstrap = (m-1) S_max coupled micro RK steps of size h,
recording RHS values at the mesh-aligned times.  R8 the N-rate generalisation:

  mesh g steps every s_g finest micro steps (h_g = s_g h, H = S_max h) and keeps base_g (its
  state at t_g) and ring_g (R at t_g - (m-1) h_g, ..., t_g).  For j = 1..S_max:
    1. every mesh: y_g = base_g + h_g sum_k w_k R_{g,k},  w = weights over [0, theta],
       theta = (t + j h - t_g)/h_g  (full AB step when theta = 1, partial otherwise)
    2. meshes with j mod s_g == 0: R_g = RHS_g(all y) at t + j h
    3. for those: push R_g into ring_g, base_g <- y_g, t_g <- t + j h.
SRAB (single-rate AB) is the same code with every s_g = 1.
macro_step_var(H): the same with a macro step that changes from step to step.
macro_step_sf(reextrap): the two-rate slowest-first variants of P:536-548 (reading R-SF).
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np

from . import abcoef, rhs as rhs_mod

HEUN3 = dict(c=(0, Fr(1, 3), Fr(2, 3)), a=((), (Fr(1, 3),), (0, Fr(2, 3))),
             b=(Fr(1, 4), 0, Fr(3, 4)))
RK4 = dict(c=(0, Fr(1, 2), Fr(1, 2), 1), a=((), (Fr(1, 2),), (0, Fr(1, 2)), (0, 0, 1)),
           b=(Fr(1, 6), Fr(1, 3), Fr(1, 3), Fr(1, 6)))


def rk_tableau(order_n):
    return RK4 if order_n >= 4 else HEUN3


def rk_step(rhs_fn, states, h, tab, on_first_stage=None, counts=None):
    """One explicit RK step of the coupled system; rhs_fn(states, which=None) -> list.
    `on_first_stage(k1)` sees the stage-1 RHS (the RHS at the step's start state)."""
    G = len(states)
    ks = []
    for s in range(len(tab["b"])):
        y = [states[g].copy() for g in range(G)]
        for j, a in enumerate(tab["a"][s]):
            if a != 0:
                for g in range(G):
                    y[g] = y[g] + (h * float(a)) * ks[j][g]
        k = rhs_fn(y)
        if counts is not None:
            for g in range(G):
                counts[g] += 1
        if s == 0 and on_first_stage is not None:
            on_first_stage(k)
        ks.append(k)
    out = []
    for g in range(G):
        y = states[g].copy()
        for j, b in enumerate(tab["b"]):
            if b != 0:
                y = y + (h * float(b)) * ks[j][g]
        out.append(y)
    return out


class MRAB:
    """Oracle integrator state.  `steps` = step multiples s_g (default: the problem's)."""

    def __init__(self, problem, setup=None, steps=None, rhs_fn=None):
        """`rhs_fn(states, which=None)` overrides the PDE right-hand side (used by the
        linear-ODE pins); by default the coupled SBP-SAT RHS of oracle.rhs."""
        self.p = problem
        if rhs_fn is None:
            self.setup = setup if setup is not None else rhs_mod.build(problem)
            rhs_fn = lambda st, which=None: rhs_mod.rhs(problem, self.setup, st, which)  # noqa
        self.rhs_fn = rhs_fn
        self.s = list(steps) if steps is not None else [m.step_multiple for m in problem.meshes]
        self.S = max(self.s)
        self.m = problem.history_m
        self.n = problem.order_n
        self.h = problem.h
        G = len(problem.meshes)
        self.base = [q.astype(np.float64).copy() for q in problem.q0]
        self.rings = [[] for _ in range(G)]          # oldest first
        self.tg = [Fr(0)] * G                        # in units of h
        self.t = Fr(0)
        self.counts = [0] * G
        self.macro = 0
        self._w = {}
        self.rtimes = None                           # variable-step mode: history node times
        self.time = None
        self.tgp = None

    def weights(self, theta):
        key = Fr(theta)
        if key not in self._w:
            self._w[key] = [float(x) for x in abcoef.partial_weights(self.m, self.n, key)]
        return self._w[key]

    def bootstrap(self):
        """(m-1) S coupled micro RK steps; rings then hold m-1 entries; the RHS at the end of
        the bootstrap is evaluated here too, completing them."""
        G = len(self.base)
        tab = rk_tableau(self.n)
        nsteps = (self.m - 1) * self.S
        y = self.base
        for k in range(nsteps):
            def rec(k1, k=k):
                for g in range(G):
                    left = nsteps - k          # micro steps until the end of the bootstrap
                    if left % self.s[g] == 0 and left // self.s[g] <= self.m - 1:
                        self.rings[g].append(k1[g])
            y = rk_step(self.rhs_fn, y, self.h, tab, rec, self.counts)
        self.base = y
        self.t = Fr(nsteps)
        self.tg = [self.t] * G
        R = self.rhs_fn(self.base)
        for g in range(G):
            self.rings[g].append(R[g])
            self.counts[g] += 1
            assert len(self.rings[g]) == self.m

    def macro_step(self):
        if self.rtimes is not None:                  # after variable steps: nodes are not uniform
            return self.macro_step_var(self.S * Fr(self.h))
        G = len(self.base)
        for j in range(1, self.S + 1):
            tj = self.t + j
            ys = []
            for g in range(G):
                theta = (tj - self.tg[g]) / self.s[g]
                w = self.weights(theta)
                hg = self.h * self.s[g]
                y = self.base[g].copy()
                for wk, Rk in zip(w, self.rings[g]):
                    y = y + (hg * wk) * Rk
                ys.append(y)
            stepping = [g for g in range(G) if j % self.s[g] == 0]
            R = self.rhs_fn(ys, which=stepping)
            for g in stepping:
                self.rings[g] = self.rings[g][1:] + [R[g]]
                self.base[g] = ys[g]
                self.tg[g] = tj
                self.counts[g] += 1
        self.t = self.t + self.S
        self.macro += 1

    def macro_step_var(self, H):
        """One macro step of size H (physical time) with h = H / S_max: "The macro-timestep
        H_i can change on a per-macrostep basis, with the micro-timestep h_i defined such that
        h_i = H_i/SR".  The history values of a mesh then sit at non-uniform times,
        so the weights of every (partial) integral come from eq:vandermonde with
        the actual node times: y_g = base_g + sum_k w_k R_{g,k}, w = ab_weights(nodes - t_g,
        n, 0, t + j h - t_g) (physical time units; reduces to macro_step for constant H)."""
        G = len(self.base)
        if self.rtimes is None:
            h0 = Fr(self.h)
            self.time = h0 * self.t
            self.rtimes = [[self.time - (self.m - 1 - k) * self.s[g] * h0 for k in range(self.m)]
                           for g in range(G)]
            self.tgp = [self.time] * G
        h = Fr(H) / self.S
        for j in range(1, self.S + 1):
            tj = self.time + j * h
            ys = []
            for g in range(G):
                nodes = [tau - self.tgp[g] for tau in self.rtimes[g]]
                w = abcoef.ab_weights(nodes, self.n, 0, tj - self.tgp[g])
                y = self.base[g].copy()
                for wk, Rk in zip(w, self.rings[g]):
                    y = y + float(wk) * Rk
                ys.append(y)
            stepping = [g for g in range(G) if j % self.s[g] == 0]
            R = self.rhs_fn(ys, which=stepping)
            for g in stepping:
                self.rings[g] = self.rings[g][1:] + [R[g]]
                self.rtimes[g] = self.rtimes[g][1:] + [tj]
                self.base[g] = ys[g]
                self.tgp[g] = tj
                self.counts[g] += 1
        self.time = self.time + Fr(H)
        self.macro += 1

    def macro_step_sf(self, reextrap=False):
        """Two-rate slowest-first macro step ("an algorithm in which the slow
        component is instead advanced first", with "the choice of whether or not to
        re-extrapolate the slow state after additional state and right-hand side information is
        gathered at the micro-timestep level"; the paper gives no steps, reading R-SF of
        DESIGN.md §2, after [gear1984multirate]).  Meshes with s_g = S are slow, s_g = 1 fast.
          1. slow: y_s(t+H) = s(t) + H sum_k alpha_k R_{s,k}  (the AB step);
             fast, extrapolated over the whole macro step: f~(t+H) = f(t) + h sum_k w_k(S) R_{f,k};
          2. R_s(t+H) = a_s(f~(t+H), y_s(t+H))  -- the slow component is evaluated first;
          3. for j = 1..S: f(t+jh) by its AB step; the slow state the fast RHS sees at t + j h,
             j < S, is s(t) + H * (partial integral over [0, j/S] of the slow extrapolant):
               reextrap = False: the extrapolant of Step 1 (history up to t);
               reextrap = True : re-formed with R_s(t+H) as its newest node (nodes
                                 -(m-2), ..., 0, 1 in units of H), i.e. an interpolant;
             at j = S it is y_s(t+H); evaluate a_f, push;
          4. push R_s(t+H), s(t+H) = y_s(t+H)."""
        G = len(self.base)
        S = self.S
        slow = [g for g in range(G) if self.s[g] == S]
        fast = [g for g in range(G) if self.s[g] == 1]
        if S == 1 or len(slow) + len(fast) != G:
            raise ValueError("slowest-first is defined here for two rates (1 and S > 1)")
        H = self.h * S
        m, n = self.m, self.n
        nodes = abcoef.uniform_nodes(m)
        w_full = [float(x) for x in abcoef.ab_weights(nodes, n, 0, 1)]
        w_long = [float(x) for x in abcoef.ab_weights(nodes, n, 0, S)]

        def comb(g, step, w, hist):
            y = self.base[g].copy()
            for wk, Rk in zip(w, hist):
                y = y + (step * wk) * Rk
            return y
        ys = [None] * G
        for g in slow:
            ys[g] = comb(g, H, w_full, self.rings[g])
        for g in fast:
            ys[g] = comb(g, self.h, w_long, self.rings[g])
        Rs = self.rhs_fn(ys, which=slow)
        y_slow_end = {g: ys[g] for g in slow}
        for g in slow:
            self.counts[g] += 1
        for j in range(1, S + 1):
            ys = [None] * G
            for g in fast:
                ys[g] = comb(g, self.h, w_full, self.rings[g])
            for g in slow:
                if j == S:
                    ys[g] = y_slow_end[g]
                elif reextrap:
                    nd = [Fr(-(m - 2) + k) for k in range(m)]          # ..., 0, 1
                    w = [float(x) for x in abcoef.ab_weights(nd, n, 0, Fr(j, S))]
                    ys[g] = comb(g, H, w, self.rings[g][1:] + [Rs[g]])
                else:
                    w = [float(x) for x in abcoef.ab_weights(nodes, n, 0, Fr(j, S))]
                    ys[g] = comb(g, H, w, self.rings[g])
            R = self.rhs_fn(ys, which=fast)
            for g in fast:
                self.rings[g] = self.rings[g][1:] + [R[g]]
                self.base[g] = ys[g]
                self.counts[g] += 1
        for g in slow:
            self.rings[g] = self.rings[g][1:] + [Rs[g]]
            self.base[g] = y_slow_end[g]
        self.t = self.t + S
        self.tg = [self.t] * G
        self.macro += 1

    def run(self, n_macro, scheme="fastest_first"):
        if not self.rings[0]:
            self.bootstrap()
        if scheme != "fastest_first":
            for _ in range(n_macro):
                self.macro_step_sf(reextrap=(scheme == "slowest_first_reextrap"))
            return self.base
        for _ in range(n_macro):
            self.macro_step()
        return self.base
