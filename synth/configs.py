"""The five synthetic overset workloads of BASELINE.json (`configs[0..4]`) and reduced-size
variants of each ("test" scale) that the oracle finishes in seconds.

Every array here is fp64.  Layout conventions shared by all consumers:
  * a mesh has `shape = (n0, n1[, n2])` in INDEX order (i fastest);
  * coordinates `xyz` have numpy shape (d, n_{d-1}, ..., n0) (C order => i fastest);
  * a state has numpy shape (nc, n_{d-1}, ..., n0) with nc = d + 2 components
    (rho, rho*u_1..rho*u_d, rho*E).
Boundary tags per face: OVERSET / FARFIELD / WALL / PERIODIC.

Sources of every number: BASELINE.json `configs` strings, SURVEY.md §8(d) (the table of the
synthetic recipe, incl. the finest micro step h of each config computed there from the
eq:ts reading G20), PAPER.md P:1646-1653 (isentropic vortex).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

OVERSET, FARFIELD, WALL, PERIODIC = 0, 1, 2, 3

GAMMA = 1.4


@dataclass
class Mesh:
    name: str
    shape: Tuple[int, ...]            # (n0, n1[, n2]) index order
    xyz: np.ndarray                   # (d, n_{d-1}, ..., n0)
    periodic: Tuple[bool, ...]
    face_bc: Tuple[Tuple[int, int], ...]   # per direction (lo, hi)
    priority: int
    step_multiple: int
    # per direction: the coordinate jump across the periodic seam, x(i + n) = x(i) + period[k]
    # (zeros for non-periodic directions and for closed curves such as the O-grid)
    period: Tuple[Tuple[float, ...], ...] = None

    def __post_init__(self):
        if self.period is None:
            d = len(self.shape)
            self.period = tuple(tuple(0.0 for _ in range(d)) for _ in range(d))

    @property
    def dim(self):
        return len(self.shape)

    @property
    def npts(self):
        return int(np.prod(self.shape))


@dataclass
class Problem:
    name: str
    dim: int
    meshes: List[Mesh]
    q0: List[np.ndarray]
    gamma: float = GAMMA
    Re: float = 0.0
    Pr: float = 0.72
    viscous: bool = False
    q_inf: np.ndarray = None
    wall_T: float = 1.0
    order_n: int = 3
    history_m: int = 3
    h: float = 1e-3                   # finest micro step
    n_macro: int = 1                  # macro steps the workload runs (after bootstrap)
    notes: dict = field(default_factory=dict)

    @property
    def nc(self):
        return self.dim + 2

    @property
    def s_max(self):
        return max(m.step_multiple for m in self.meshes)


def primitive_to_conserved(rho, vel, p, gamma=GAMMA):
    """(rho, u_i, p) -> (rho, rho u_i, rho E) with rho E = p/(gamma-1) + rho|u|^2/2."""
    vel = [np.asarray(v, dtype=np.float64) for v in vel]
    rho = np.asarray(rho, dtype=np.float64)
    ke = 0.5 * rho * sum(v * v for v in vel)
    return np.stack([rho * np.ones_like(vel[0])] + [rho * v for v in vel]
                    + [p / (gamma - 1.0) + ke]).astype(np.float64)


def _axis_coords(lo, hi, n, periodic):
    if periodic:
        return lo + np.arange(n, dtype=np.float64) * ((hi - lo) / n)
    return lo + np.arange(n, dtype=np.float64) * ((hi - lo) / (n - 1))


def _cart(name, lows, highs, shape, periodic, face_bc, priority, s):
    d = len(shape)
    axes = [_axis_coords(lows[k], highs[k], shape[k], periodic[k]) for k in range(d)]
    # meshgrid in numpy order (n_{d-1}, ..., n0)
    grids = np.meshgrid(*[axes[k] for k in reversed(range(d))], indexing="ij")
    xyz = np.stack([grids[d - 1 - k] for k in range(d)]).astype(np.float64)
    period = tuple(tuple((highs[k] - lows[k]) if (periodic[k] and c == k) else 0.0
                         for c in range(d)) for k in range(d))
    return Mesh(name, tuple(shape), np.ascontiguousarray(xyz), tuple(periodic),
                tuple(tuple(f) for f in face_bc), priority, s, period)


def _logical(shape):
    d = len(shape)
    axes = [np.arange(shape[k], dtype=np.float64) / (shape[k] - 1) for k in range(d)]
    grids = np.meshgrid(*[axes[k] for k in reversed(range(d))], indexing="ij")
    return [grids[d - 1 - k] for k in range(d)]


def _uniform_state(mesh, rho, vel, p, gamma=GAMMA):
    shp = tuple(reversed(mesh.shape))
    return primitive_to_conserved(np.full(shp, rho), [np.full(shp, v) for v in vel],
                                  np.full(shp, p), gamma)


def _qinf(dim, u, gamma=GAMMA):
    vel = [u] + [0.0] * (dim - 1)
    return primitive_to_conserved(np.array(1.0), [np.array(v) for v in vel],
                                  np.array(1.0 / gamma), gamma).reshape(dim + 2)


# ---------------------------------------------------------------------------------------
# config 1: 2-D Euler isentropic vortex, two Cartesian meshes
# ---------------------------------------------------------------------------------------
def _vortex_state(mesh, omega=5.0, phi=1.0, x0=0.0, y0=0.0, u0=0.5, v0=0.0, c0=1.0, t=0.0,
                  gamma=GAMMA):
    """Convecting vortex of P:1646-1653 with p = rho^gamma / gamma (nondim c_inf = 1)."""
    x, y = mesh.xyz[0], mesh.xyz[1]
    dx, dy = x - x0 - u0 * t, y - y0 - v0 * t
    r2 = dx * dx + dy * dy
    rho = (1.0 - omega ** 2 * (gamma - 1.0) / (8.0 * math.pi ** 2 * c0 ** 2)
           * np.exp(1.0 - phi ** 2 * r2)) ** (1.0 / (gamma - 1.0))
    u = u0 - omega / (2 * math.pi) * phi * dy * np.exp(0.5 * (1.0 - phi ** 2 * r2))
    v = v0 + omega / (2 * math.pi) * phi * dx * np.exp(0.5 * (1.0 - phi ** 2 * r2))
    p = rho ** gamma / gamma
    return primitive_to_conserved(rho, [u, v], p, gamma)


def config1(scale="full", order_n=3, history_m=None, sr=4, n_macro=None):
    n_bg, n_in = (41, 41)
    if scale == "tiny":
        n_bg, n_in = 41, 41
    bg = _cart("background", (-5.0, -5.0), (5.0, 5.0), (n_bg, n_bg), (False, False),
               ((FARFIELD, FARFIELD), (FARFIELD, FARFIELD)), 0, sr)
    inner = _cart("inner", (-1.25, -1.25), (1.25, 1.25), (n_in, n_in), (False, False),
                  ((OVERSET, OVERSET), (OVERSET, OVERSET)), 1, 1)
    meshes = [bg, inner]
    q0 = [_vortex_state(m) for m in meshes]
    return Problem("config1", 2, meshes, q0, viscous=False, Re=0.0, q_inf=_qinf(2, 0.5),
                   order_n=order_n, history_m=history_m or order_n, h=8.91e-3,
                   n_macro=n_macro if n_macro is not None else (200 if scale == "full" else 20),
                   notes={"workload": "2D Euler isentropic vortex, bg 41^2 + inner 41^2"})


# ---------------------------------------------------------------------------------------
# config 2: 2-D NS pressure pulse, Cartesian bg + rotated, sinusoidally perturbed inner
# ---------------------------------------------------------------------------------------
def _inner_curvilinear_2d(name, n, side, amp, angle_deg, priority, s):
    xi, eta = _logical((n, n))
    a = math.radians(angle_deg)
    X0 = side * (xi - 0.5)
    Y0 = side * (eta - 0.5)
    bump = amp * np.sin(2 * math.pi * xi) * np.sin(2 * math.pi * eta)
    x = math.cos(a) * X0 - math.sin(a) * Y0 + bump
    y = math.sin(a) * X0 + math.cos(a) * Y0 + bump
    xyz = np.ascontiguousarray(np.stack([x, y]))
    return Mesh(name, (n, n), xyz, (False, False), ((OVERSET, OVERSET), (OVERSET, OVERSET)),
                priority, s)


def _pulse_state(mesh, u, amp, width, dim, gamma=GAMMA):
    r2 = sum(mesh.xyz[k] ** 2 for k in range(dim))
    p = 1.0 / gamma + amp * np.exp(-r2 / width ** 2)
    vel = [np.full_like(r2, u)] + [np.zeros_like(r2) for _ in range(dim - 1)]
    return primitive_to_conserved(np.ones_like(r2), vel, p, gamma)


def config2(scale="full", order_n=3, history_m=None, sr=4, n_macro=None):
    if scale == "full":
        n_bg, L, n_in, h, nm = 401, 10.0, 201, 1.5e-3, 1000
    else:
        n_bg, L, n_in, h, nm = 61, 3.0, 41, 6.0e-3, 6
    bg = _cart("background", (-L, -L), (L, L), (n_bg, n_bg), (False, False),
               ((FARFIELD, FARFIELD), (FARFIELD, FARFIELD)), 0, sr)
    inner = _inner_curvilinear_2d("inner", n_in, 2.5, 0.05, 30.0, 1, 1)
    meshes = [bg, inner]
    q0 = [_pulse_state(m, 0.3, 0.01, 0.2, 2) for m in meshes]
    return Problem("config2", 2, meshes, q0, viscous=True, Re=1000.0, Pr=0.72,
                   q_inf=_qinf(2, 0.3), order_n=order_n, history_m=history_m or order_n,
                   h=h, n_macro=n_macro if n_macro is not None else nm,
                   notes={"workload": f"2D NS pulse, bg {n_bg}^2 + curvilinear inner {n_in}^2"})


# ---------------------------------------------------------------------------------------
# config 3: 2-D viscous cylinder, O-grid (wall) + Cartesian background
# ---------------------------------------------------------------------------------------
def _ogrid(name, n_theta, n_r, r0, r1, stretch, priority, s):
    j = np.arange(n_r, dtype=np.float64)
    dr0 = (r1 - r0) * (stretch - 1.0) / (stretch ** (n_r - 1) - 1.0)
    r = r0 + dr0 * (stretch ** j - 1.0) / (stretch - 1.0)
    r[-1] = r1
    th = -2.0 * math.pi * np.arange(n_theta, dtype=np.float64) / n_theta   # clockwise
    R, TH = np.meshgrid(r, th, indexing="ij")          # numpy order (n_r, n_theta)
    xyz = np.ascontiguousarray(np.stack([R * np.cos(TH), R * np.sin(TH)]))
    return Mesh(name, (n_theta, n_r), xyz, (True, False),
                ((PERIODIC, PERIODIC), (WALL, OVERSET)), priority, s)


def config3(scale="full", order_n=3, history_m=None, sr=4, n_macro=None):
    if scale == "full":
        nt, nr, n_bg, L, h, nm = 512, 128, 1024, 20.0, 5.41e-7, 100
    else:
        nt, nr, n_bg, L, h, nm = 96, 24, 61, 3.0, 2.0e-4, 6
    og = _ogrid("ogrid", nt, nr, 0.5, 2.0, 1.05, 1, 1)
    bg = _cart("background", (-L, -L), (L, L), (n_bg, n_bg), (False, False),
               ((FARFIELD, FARFIELD), (FARFIELD, FARFIELD)), 0, sr)
    meshes = [og, bg]
    rng = np.random.default_rng(3)
    q0 = []
    for m in meshes:
        shp = tuple(reversed(m.shape))
        prim = []
        for base in (1.0, 0.2, 0.0, 1.0 / GAMMA):
            prim.append(base + 1e-4 * rng.uniform(-1.0, 1.0, size=shp))
        q0.append(primitive_to_conserved(prim[0], prim[1:3], prim[3]))
    return Problem("config3", 2, meshes, q0, viscous=True, Re=200.0, Pr=0.72,
                   q_inf=_qinf(2, 0.2), wall_T=1.0, order_n=order_n,
                   history_m=history_m or order_n, h=h,
                   n_macro=n_macro if n_macro is not None else nm,
                   notes={"workload": f"2D cylinder, O-grid {nt}x{nr} + bg {n_bg}^2, SR {sr}"})


# ---------------------------------------------------------------------------------------
# config 4: 3-D NS, periodic(y,z) background + refined Cartesian block
# ---------------------------------------------------------------------------------------
def config4(scale="full", order_n=3, history_m=None, sr=4, n_macro=None):
    if scale == "full":
        n_bg, L, n_b, B, h, nm = 256, 8.0, 192, 1.5, 1.01e-3, 100
    else:
        n_bg, L, n_b, B, h, nm = 36, 3.6, 26, 1.0, 6.0e-3, 4
    bg = _cart("background", (-L, -L, -L), (L, L, L), (n_bg, n_bg, n_bg), (False, True, True),
               ((FARFIELD, FARFIELD), (PERIODIC, PERIODIC), (PERIODIC, PERIODIC)), 0, sr)
    blk = _cart("block", (-B, -B, -B), (B, B, B), (n_b, n_b, n_b), (False, False, False),
                ((OVERSET, OVERSET),) * 3, 1, 1)
    meshes = [bg, blk]
    q0 = [_pulse_state(m, 0.3, 0.01, 0.3, 3) for m in meshes]
    return Problem("config4", 3, meshes, q0, viscous=True, Re=500.0, Pr=0.72,
                   q_inf=_qinf(3, 0.3), order_n=order_n, history_m=history_m or order_n,
                   h=h, n_macro=n_macro if n_macro is not None else nm,
                   notes={"workload": f"3D NS pulse, bg {n_bg}^3 + block {n_b}^3"})


# ---------------------------------------------------------------------------------------
# config 5: 3-D four nested meshes, rates 1:2:4:8, two warped
# ---------------------------------------------------------------------------------------
def _nested_mesh(name, n, hk, warp, priority, s):
    ext = (n - 1) * hk
    m = _cart(name, (-ext / 2,) * 3, (ext / 2,) * 3, (n, n, n), (False,) * 3,
              ((OVERSET, OVERSET),) * 3, priority, s)
    if warp:
        xi, eta, zeta = _logical((n, n, n))
        bump = warp * ext * np.sin(2 * math.pi * xi) * np.sin(2 * math.pi * eta) \
            * np.sin(2 * math.pi * zeta)
        m.xyz = np.ascontiguousarray(m.xyz + bump[None])
    return m


def _config5_velocity(meshes, coarse, rng, nmodes=32, rms=1e-3):
    ks = []
    while len(ks) < nmodes:
        k = rng.integers(-4, 5, size=3)
        n2 = float(np.dot(k, k))
        if 1.0 <= math.sqrt(n2) <= 4.0:
            ks.append(k.astype(np.float64))
    ks = np.array(ks)
    phases = rng.uniform(0.0, 2 * math.pi, size=(nmodes, 3))

    def raw(mesh):
        # sum_m cos(pi k_m.(x+1) + phi_mc) = Re sum_m exp(i pi k_m.(x+1)) exp(i phi_mc)
        acc = [np.zeros(mesh.xyz.shape[1:]) for _ in range(3)]
        for mi in range(nmodes):
            arg = math.pi * sum(ks[mi, a] * (mesh.xyz[a] + 1.0) for a in range(3))
            E = np.exp(1j * arg)
            for c in range(3):
                acc[c] += (E * complex(math.cos(phases[mi, c]), math.sin(phases[mi, c]))).real
        return acc

    rc = raw(coarse)
    amps = [rms / math.sqrt(float(np.mean(rc[c] ** 2))) for c in range(3)]
    return [[amps[c] * r for c, r in enumerate(rc if m is coarse else raw(m))] for m in meshes]


def config5(scale="full", order_n=4, history_m=None, sr=None, n_macro=None):
    if scale == "full":
        n, h, nm = 160, 2.52e-5, 50
    else:
        n, h, nm = 32, 4.0e-4, 2
    h3 = 2.0 / n
    meshes = []
    for k in range(3):
        hk = h3 / 2 ** (3 - k)
        meshes.append(_nested_mesh(f"level{k}", n, hk, 0.03 if k < 2 else 0.0, 3 - k, 2 ** k))
    coarse = _cart("level3", (-1.0,) * 3, (1.0,) * 3, (n, n, n), (True,) * 3,
                   ((PERIODIC, PERIODIC),) * 3, 0, 8)
    meshes.append(coarse)
    rng = np.random.default_rng(5)
    vels = _config5_velocity(meshes, coarse, rng)
    q0 = []
    for m, v in zip(meshes, vels):
        shp = m.xyz.shape[1:]
        q0.append(primitive_to_conserved(np.ones(shp), [0.4 + v[0], v[1], v[2]],
                                         np.full(shp, 1.0 / GAMMA)))
    return Problem("config5", 3, meshes, q0, viscous=True, Re=1000.0, Pr=0.72,
                   q_inf=_qinf(3, 0.4), order_n=order_n, history_m=history_m or order_n,
                   h=h, n_macro=n_macro if n_macro is not None else nm,
                   notes={"workload": f"3D 4 nested {n}^3, rates 1:2:4:8"})


_BUILDERS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def config_names():
    return sorted(_BUILDERS)


def make_config(cid: int, scale: str = "full", **kw) -> Problem:
    """Build workload `cid` (1..5) at `scale` in {"full", "test"}."""
    return _BUILDERS[cid](scale=scale, **kw)


# ---------------------------------------------------------------------------------------
# pin workloads (App. C of the paper): inputs only, expected values live in the tests
# ---------------------------------------------------------------------------------------
def mms_box_in_box(N, kind="inviscid", gamma=GAMMA):
    """outer [-1,1]^2 periodic with N x N points, inner [-0.5,0.5]^2 with
    (N+1)/2 x (N+1)/2 points (reading G27), SAT interpolation between them.
    inviscid: rho = 1, rho u = sin(2 pi (x - 1/2)), rho v = 0
    viscous : rho = 1, rho u = sin(2 pi (y - 1/2)), rho v = 0, Re = 1
    p = 1/gamma in both (the paper leaves p free)."""
    outer = _cart("outer", (-1.0, -1.0), (1.0, 1.0), (N, N), (True, True),
                  ((PERIODIC, PERIODIC), (PERIODIC, PERIODIC)), 0, 1)
    ni = (N + 1) // 2
    inner = _cart("inner", (-0.5, -0.5), (0.5, 0.5), (ni, ni), (False, False),
                  ((OVERSET, OVERSET), (OVERSET, OVERSET)), 1, 1)
    q0 = []
    for m in (outer, inner):
        x, y = m.xyz
        arg = x if kind == "inviscid" else y
        u = np.sin(2 * math.pi * (arg - 0.5))
        q0.append(primitive_to_conserved(np.ones_like(x), [u, np.zeros_like(x)],
                                         np.full_like(x, 1.0 / gamma), gamma))
    visc = kind != "inviscid"
    return Problem(f"mms_{kind}_{N}", 2, [outer, inner], q0, viscous=visc,
                   Re=1.0 if visc else 0.0, Pr=0.72, q_inf=_qinf(2, 0.0))


def vortex_box_in_box(N, omega=2.0, phi=8.0, u0=2.0, gamma=GAMMA):
    """outer [-1,1]x[-0.5,0.5] periodic, inner [-0.38,0.38]^2, both N x N,
    convecting vortex with bulk velocity (2, 0) (omega, phi: reading, not printed)."""
    outer = _cart("outer", (-1.0, -0.5), (1.0, 0.5), (N, N), (True, True),
                  ((PERIODIC, PERIODIC), (PERIODIC, PERIODIC)), 0, 1)
    inner = _cart("inner", (-0.38, -0.38), (0.38, 0.38), (N, N), (False, False),
                  ((OVERSET, OVERSET), (OVERSET, OVERSET)), 1, 1)
    q0 = [_vortex_state(m, omega=omega, phi=phi, u0=u0) for m in (outer, inner)]
    return Problem(f"vortex_{N}", 2, [outer, inner], q0, viscous=False,
                   q_inf=_qinf(2, u0), notes=dict(omega=omega, phi=phi, u0=u0))


def vortex_exact(mesh, t, omega=2.0, phi=8.0, u0=2.0, period_x=2.0, gamma=GAMMA):
    """Exact translating vortex at time t, periodic images in x summed over
    the nearest centre (the vortex is compact at these parameters)."""
    xc = ((u0 * t + 1.0) % period_x) - 1.0
    return _vortex_state(mesh, omega=omega, phi=phi, x0=xc, u0=0.0, gamma=gamma)
