"""Thin ctypes binding of libmrab.so (include/mrab.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the
library is missing this module raises at import of the symbol table.

Names mirror the C ABI: `ab_weights`, `Plan` (mrab_plan_*), `Context` (mrab_create /
mrab_step / mrab_get_state / mrab_set_state / mrab_rhs / mrab_get_counters).  PyTorch is used
only for the device workspace and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmrab.so")

STATUS = {0: "OK", 1: "INVALID", 2: "DEGENERATE_NODES", 3: "INSUFFICIENT_HISTORY",
          4: "MISALIGNED", 5: "ORPHAN", 6: "SEGMENT", 7: "NONFINITE", 8: "CUDA", 9: "WORKSPACE"}


class MrabError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


class MeshDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int * 3), ("periodic", C.c_int * 3),
                ("face_bc", (C.c_int * 2) * 3), ("period", (C.c_double * 3) * 3),
                ("xyz", C.POINTER(C.c_double)), ("priority", C.c_int),
                ("step_multiple", C.c_int), ("metrics", C.POINTER(C.c_double)),
                ("iblank", C.POINTER(C.c_int8))]


class Donor(C.Structure):
    """mrab_donor: one receiver and its donor stencil (include/mrab.h)."""
    _fields_ = [("recv_mesh", C.c_int32), ("donor_mesh", C.c_int32), ("recv_index", C.c_int64),
                ("base", C.c_int32 * 3), ("reserved", C.c_int32), ("w", (C.c_double * 4) * 3)]


DONOR_DTYPE = np.dtype([("recv_mesh", "<i4"), ("donor_mesh", "<i4"), ("recv_index", "<i8"),
                        ("base", "<i4", (3,)), ("reserved", "<i4"), ("w", "<f8", (3, 4))])
assert DONOR_DTYPE.itemsize == C.sizeof(Donor)


class ProblemDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_meshes", C.c_int), ("meshes", C.POINTER(MeshDesc)),
                ("gamma", C.c_double), ("Re", C.c_double), ("Pr", C.c_double),
                ("viscous", C.c_int), ("q_inf", C.c_double * 5), ("wall_T", C.c_double),
                ("order_n", C.c_int), ("history_m", C.c_int), ("h", C.c_double),
                ("n_donors", C.c_int64), ("donors", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MrabError(1, f"{LIB_PATH} not built (run paper_1805_06607_b200/build.py)")
        L = C.CDLL(LIB_PATH)
        vp, i64p = C.c_void_p, C.POINTER(C.c_int64)
        dp = C.POINTER(C.c_double)
        L.mrab_ab_weights.argtypes = [dp, C.c_int, C.c_int, C.c_double, C.c_double, dp]
        L.mrab_plan_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(vp)]
        L.mrab_plan_destroy.argtypes = [vp]
        L.mrab_plan_destroy.restype = None
        L.mrab_plan_info.argtypes = [vp, C.c_int, i64p, i64p, i64p]
        L.mrab_plan_get_tables.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
        L.mrab_plan_get_metrics.argtypes = [vp, C.c_int, vp, vp]
        L.mrab_plan_get_face_flags.argtypes = [vp, C.c_int, vp]
        L.mrab_overset_build.argtypes = [C.POINTER(ProblemDesc), C.POINTER(vp), C.POINTER(vp),
                                         i64p]
        L.mrab_free.argtypes = [vp]
        L.mrab_free.restype = None
        L.mrab_workspace_bytes.argtypes = [vp]
        L.mrab_workspace_bytes.restype = C.c_size_t
        L.mrab_create.argtypes = [vp, C.POINTER(vp), vp, C.c_size_t, vp, C.POINTER(vp)]
        L.mrab_destroy.argtypes = [vp]
        L.mrab_destroy.restype = None
        L.mrab_step.argtypes = [vp, C.c_int]
        L.mrab_step_h.argtypes = [vp, C.c_int, C.c_double]
        L.mrab_step_scheme.argtypes = [vp, C.c_int, C.c_int]
        L.mrab_rk_step.argtypes = [vp, C.c_int, C.c_int, C.c_double]
        L.mrab_partition.argtypes = [vp, C.c_int, C.POINTER(C.c_int), dp]
        L.mrab_dist_unique_id.argtypes = [vp]
        L.mrab_dist_attach.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.mrab_dist_stats.argtypes = [vp, i64p, i64p]
        L.mrab_dt.argtypes = [vp, dp]
        L.mrab_step_cfl.argtypes = [vp, C.c_int, C.c_double, dp]
        L.mrab_get_state.argtypes = [vp, C.c_int, vp, dp]
        L.mrab_set_state.argtypes = [vp, C.c_int, vp]
        L.mrab_get_history.argtypes = [vp, C.c_int, C.c_int, vp]
        L.mrab_set_history.argtypes = [vp, C.c_int, C.c_int, vp]
        L.mrab_rhs.argtypes = [vp, C.POINTER(vp), C.POINTER(vp)]
        L.mrab_get_counters.argtypes = [vp, i64p, i64p, i64p]
        L.mrab_launches_per_macro_step.argtypes = [vp, i64p]
        L.mrab_time_kernel.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp]
        L.mrab_set_trace.argtypes = [vp, vp]
        L.mrab_last_error.restype = C.c_char_p
        for name in ("mrab_ab_weights", "mrab_plan_create", "mrab_plan_info",
                     "mrab_plan_get_tables", "mrab_plan_get_metrics", "mrab_create",
                     "mrab_step", "mrab_get_state", "mrab_set_state", "mrab_rhs",
                     "mrab_get_history", "mrab_set_history", "mrab_get_counters",
                     "mrab_launches_per_macro_step", "mrab_time_kernel", "mrab_step_h", "mrab_dt", "mrab_step_scheme", "mrab_rk_step", "mrab_partition", "mrab_dist_unique_id", "mrab_dist_attach",
                     "mrab_dist_stats", "mrab_step_cfl"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


EXPORTED = ["mrab_ab_weights", "mrab_plan_create", "mrab_plan_destroy", "mrab_plan_info",
            "mrab_plan_get_tables", "mrab_plan_get_metrics", "mrab_workspace_bytes",
            "mrab_create", "mrab_destroy", "mrab_step", "mrab_get_state", "mrab_set_state",
            "mrab_rhs", "mrab_get_counters", "mrab_launches_per_macro_step", "mrab_time_kernel",
            "mrab_set_trace", "mrab_last_error", "mrab_get_history", "mrab_set_history",
            "mrab_overset_build", "mrab_free", "mrab_plan_get_face_flags", "mrab_step_h", "mrab_dt", "mrab_step_scheme", "mrab_rk_step", "mrab_partition", "mrab_dist_unique_id", "mrab_dist_attach",
            "mrab_dist_stats", "mrab_step_cfl"]


def _check(st):
    if st != 0:
        raise MrabError(st, lib().mrab_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _state_ptr(buf, nelem, what):
    """Device or host address of a dense fp64 state buffer of exactly `nelem` elements (numpy
    array or torch tensor, C-contiguous); anything else raises before the library copies."""
    if isinstance(buf, np.ndarray):
        ok = buf.dtype == np.float64 and buf.flags.c_contiguous and buf.size == nelem
        ptr = buf.ctypes.data
    else:
        import torch
        ok = (isinstance(buf, torch.Tensor) and buf.dtype == torch.float64
              and buf.is_contiguous() and buf.numel() == nelem)
        ptr = buf.data_ptr() if ok else 0
    if not ok:
        raise MrabError(1, f"{what}: need a C-contiguous float64 buffer of {nelem} elements")
    return C.c_void_p(ptr)


def ab_weights(nodes, n, a, b):
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    out = np.zeros(len(nodes))
    _check(lib().mrab_ab_weights(_dptr(nodes), len(nodes), int(n), float(a), float(b),
                                 _dptr(out)))
    return out


def _problem_desc(problem, steps=None, iblank=None, metrics=None, donors=None):
    keep = []
    descs = (MeshDesc * len(problem.meshes))()
    for g, m in enumerate(problem.meshes):
        d = descs[g]
        d.dim = problem.dim
        for k in range(3):
            d.n[k] = m.shape[k] if k < problem.dim else 1
            d.periodic[k] = int(m.periodic[k]) if k < problem.dim else 0
            for s in range(2):
                d.face_bc[k][s] = int(m.face_bc[k][s]) if k < problem.dim else 3
            for c in range(3):
                d.period[k][c] = (float(m.period[k][c])
                                  if (k < problem.dim and c < problem.dim) else 0.0)
        xyz = np.ascontiguousarray(m.xyz, dtype=np.float64)
        keep.append(xyz)
        d.xyz = _dptr(xyz)
        d.priority = int(m.priority)
        d.step_multiple = int(steps[g] if steps is not None else m.step_multiple)
        npts = int(np.prod(m.shape[:problem.dim]))
        if metrics is not None and metrics[g] is not None:
            mt = np.ascontiguousarray(metrics[g], dtype=np.float64)
            assert mt.size == (1 + problem.dim ** 2) * npts, "metrics: [1 + dim^2][n...]"
            keep.append(mt)
            d.metrics = _dptr(mt)
        if iblank is not None and iblank[g] is not None:
            ib = np.ascontiguousarray(iblank[g], dtype=np.int8)
            assert ib.size == npts, "iblank: [n...]"
            keep.append(ib)
            d.iblank = ib.ctypes.data_as(C.POINTER(C.c_int8))
    pb = ProblemDesc()
    pb.dim = problem.dim
    pb.n_meshes = len(problem.meshes)
    pb.meshes = descs
    pb.gamma, pb.Re, pb.Pr = float(problem.gamma), float(problem.Re), float(problem.Pr)
    pb.viscous = int(bool(problem.viscous))
    for c in range(problem.dim + 2):
        pb.q_inf[c] = float(problem.q_inf[c])
    pb.wall_T = float(problem.wall_T)
    pb.order_n, pb.history_m = int(problem.order_n), int(problem.history_m)
    pb.h = float(problem.h)
    if donors is not None:
        dn = np.ascontiguousarray(donors, dtype=DONOR_DTYPE)
        keep.append(dn)
        pb.n_donors = len(dn)
        pb.donors = dn.ctypes.data if len(dn) else None
    return pb, keep, descs


def overset_build(problem, steps=None, iblank=None, donors=None):
    """mrab_overset_build: (list of per-mesh int8 iblank arrays, DONOR_DTYPE donor table)."""
    pb, keep, descs = _problem_desc(problem, steps, iblank, None, donors)
    ib, dn, n = C.c_void_p(), C.c_void_p(), C.c_int64()
    _check(lib().mrab_overset_build(C.byref(pb), C.byref(ib), C.byref(dn), C.byref(n)))
    try:
        sizes = [int(np.prod(m.shape[:problem.dim])) for m in problem.meshes]
        flat = np.ctypeslib.as_array(C.cast(ib, C.POINTER(C.c_int8)), (sum(sizes),)).copy()
        out_ib, o = [], 0
        for sz in sizes:
            out_ib.append(flat[o:o + sz])
            o += sz
        R = n.value
        raw = (C.c_char * (R * DONOR_DTYPE.itemsize)).from_address(dn.value) if R else b""
        table = np.frombuffer(bytes(raw), dtype=DONOR_DTYPE).copy()
    finally:
        lib().mrab_free(ib)
        lib().mrab_free(dn)
    return out_ib, table


class Plan:
    """mrab_plan: host setup.  `problem` is any object with the fields of mrab_problem
    (dim, meshes[...], gamma, Re, Pr, viscous, q_inf, wall_T, order_n, history_m, h); each
    mesh has shape, xyz, periodic, face_bc, period, priority, step_multiple."""

    def __init__(self, problem, steps=None, iblank=None, metrics=None, donors=None):
        """Optional caller-supplied setup (mrab.h): iblank[g] int8 [n...] and metrics[g]
        float64 [1 + dim^2][n...] per mesh (None entries = built by the library), donors a
        DONOR_DTYPE array (None = searched by the library)."""
        pb, self._keep, self._descs = _problem_desc(problem, steps, iblank, metrics, donors)
        h = C.c_void_p()
        _check(lib().mrab_plan_create(C.byref(pb), C.byref(h)))
        self.h = h
        self.dim = problem.dim
        self.nc = problem.dim + 2
        self.shapes = [tuple(m.shape) for m in problem.meshes]
        self.n_meshes = len(problem.meshes)
        self.history_m = int(problem.history_m)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mrab_plan_destroy(self.h)
            self.h = None

    def info(self, g):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().mrab_plan_info(self.h, g, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def tables(self, g):
        npts, _, R = self.info(g)
        ib = np.zeros(npts, np.int8)
        rp = np.zeros(max(R, 1), np.int64)
        rd = np.zeros(max(R, 1), np.int32)
        rb = np.zeros((max(R, 1), 3), np.int32)
        rw = np.zeros((max(R, 1), 3, 4))
        _check(lib().mrab_plan_get_tables(self.h, g, ib.ctypes.data, rp.ctypes.data,
                                          rd.ctypes.data, rb.ctypes.data, rw.ctypes.data))
        return dict(iblank=ib, point=rp[:R], donor=rd[:R], base=rb[:R], weights=rw[:R])

    def face_flags(self, g):
        """SAT face flags (mrab_plan_get_face_flags): bit 2k = kappa-min segment end, bit
        2k+1 = kappa-max segment end."""
        npts, _, _ = self.info(g)
        f = np.zeros(npts, np.uint8)
        _check(lib().mrab_plan_get_face_flags(self.h, g, f.ctypes.data))
        return f

    def metrics(self, g):
        npts, _, _ = self.info(g)
        jinv = np.zeros(npts)
        M = np.zeros((self.dim, self.dim, npts))
        _check(lib().mrab_plan_get_metrics(self.h, g, jinv.ctypes.data, M.ctypes.data))
        return jinv, M

    def workspace_bytes(self):
        return int(lib().mrab_workspace_bytes(self.h))


def partition(plan, nranks):
    """owner[g] and per-rank load by the work weight active points x evaluations per macro
    step (mrab_partition)."""
    G = plan.n_meshes
    ow = (C.c_int * G)()
    ld = (C.c_double * nranks)()
    _check(lib().mrab_partition(plan.h, int(nranks), ow, ld))
    return [int(x) for x in ow], [float(x) for x in ld]


class Context:
    """mrab_ctx on the current torch CUDA device and stream."""

    def __init__(self, plan: Plan, q0, stream=None, workspace=None):
        """`workspace`: optional caller-owned device buffer (torch uint8 tensor) of at least
        plan.workspace_bytes() + 256 bytes; the context uses its first 256-byte-aligned
        address."""
        import torch
        self.plan = plan
        nbytes = plan.workspace_bytes()
        if workspace is None:
            workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
        assert workspace.is_cuda and workspace.numel() >= nbytes + 256
        self.ws = workspace
        base = self.ws.data_ptr()
        off = (-base) % 256
        qs = [np.ascontiguousarray(q, dtype=np.float64) for q in q0]
        arr = (C.c_void_p * len(qs))(*[q.ctypes.data for q in qs])
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        h = C.c_void_p()
        _check(lib().mrab_create(plan.h, arr, C.c_void_p(base + off), nbytes, C.c_void_p(st),
                                 C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().mrab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    SCHEMES = {"fastest_first": 0, "slowest_first": 1, "slowest_first_reextrap": 2}

    def step(self, n_macro=1, scheme="fastest_first"):
        if scheme == "fastest_first":
            _check(lib().mrab_step(self.h, int(n_macro)))
        else:
            _check(lib().mrab_step_scheme(self.h, int(n_macro), self.SCHEMES[scheme]))

    def attach_loopback(self, world_id, rank, nranks, owner):
        """Multi-GPU test transport: this context plays `rank` of `nranks` in process-local
        world `world_id` (mrab_dist_attach, MRAB_TRANSPORT_LOOPBACK)."""
        wid = C.c_int(int(world_id))
        ow = (C.c_int * len(owner))(*[int(o) for o in owner])
        _check(lib().mrab_dist_attach(self.h, 1, C.byref(wid), int(rank), int(nranks), ow))
        self.owner, self.rank = list(owner), int(rank)

    def attach_nccl(self, dist, owner):
        """One process per GPU: rank 0 draws the NCCL unique id, torch.distributed broadcasts it,
        every rank attaches (mrab_dist_attach, MRAB_TRANSPORT_NCCL)."""
        import torch
        rank, world = dist.get_rank(), dist.get_world_size()
        buf = C.create_string_buffer(128)
        if rank == 0:
            _check(lib().mrab_dist_unique_id(buf))
        t = torch.tensor(list(buf.raw), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        raw = bytes(t.cpu().tolist())
        ow = (C.c_int * len(owner))(*[int(o) for o in owner])
        _check(lib().mrab_dist_attach(self.h, 0, C.create_string_buffer(raw, 128), rank, world, ow))
        self.owner, self.rank = list(owner), rank

    def dist_stats(self):
        b, m = C.c_int64(), C.c_int64()
        _check(lib().mrab_dist_stats(self.h, C.byref(b), C.byref(m)))
        return b.value, m.value

    def rk_step(self, h, n_steps=1, order=4):
        """n_steps coupled single-rate RK steps of size h (mrab_rk_step)."""
        _check(lib().mrab_rk_step(self.h, int(n_steps), int(order), float(h)))

    def step_h(self, H, n_macro=1):
        """n_macro MRAB macro steps of size H (variable macro step, mrab_step_h)."""
        _check(lib().mrab_step_h(self.h, int(n_macro), float(H)))

    def step_cfl(self, cfl, n_macro=1):
        """n_macro macro steps at H = cfl * S * min_g dt_g / s_g from the device estimate
        (mrab_step_cfl); returns the last H."""
        H = C.c_double()
        _check(lib().mrab_step_cfl(self.h, int(n_macro), float(cfl), C.byref(H)))
        return H.value

    def dt(self):
        """Per-mesh minimum of the eq:ts stable timestep at the current states (mrab_dt)."""
        out = (C.c_double * len(self.plan.shapes))()
        _check(lib().mrab_dt(self.h, out))
        return [float(v) for v in out]

    def get_state(self, g, out=None):
        """Copy mesh g's state into `out` (numpy array, or torch tensor on host or device)
        or a new numpy array; returns (array, t)."""
        shp = (self.plan.nc,) + tuple(reversed(self.plan.shapes[g]))
        if out is None:
            out = np.zeros(shp)
        t = C.c_double()
        _check(lib().mrab_get_state(self.h, g, _state_ptr(out, self._nelem(g), "get_state"),
                                    C.byref(t)))
        return out, t.value

    def _nelem(self, g):
        return self.plan.nc * int(np.prod(self.plan.shapes[g]))

    def set_state(self, g, src):
        _check(lib().mrab_set_state(self.h, g, _state_ptr(src, self._nelem(g), "set_state")))

    def get_history(self, g, k, out=None):
        """Committed RHS history entry k (0 = oldest of m-1) of mesh g at the macro boundary."""
        shp = (self.plan.nc,) + tuple(reversed(self.plan.shapes[g]))
        if out is None:
            out = np.zeros(shp)
        _check(lib().mrab_get_history(self.h, g, int(k),
                                      _state_ptr(out, self._nelem(g), "get_history")))
        return out

    def set_history(self, g, k, src):
        _check(lib().mrab_set_history(self.h, g, int(k),
                                      _state_ptr(src, self._nelem(g), "set_history")))

    def rhs(self, states):
        qs = [np.ascontiguousarray(q, dtype=np.float64) for q in states]
        outs = [np.zeros_like(q) for q in qs]
        a = (C.c_void_p * len(qs))(*[q.ctypes.data for q in qs])
        b = (C.c_void_p * len(qs))(*[o.ctypes.data for o in outs])
        _check(lib().mrab_rhs(self.h, a, b))
        return outs

    def counters(self):
        G = self.plan.n_meshes
        ev = np.zeros(G, np.int64)
        pr, mac = C.c_int64(), C.c_int64()
        _check(lib().mrab_get_counters(self.h, ev.ctypes.data_as(C.POINTER(C.c_int64)),
                                       C.byref(pr), C.byref(mac)))
        return ev, pr.value, mac.value

    def launches_per_macro_step(self):
        v = C.c_int64()
        _check(lib().mrab_launches_per_macro_step(self.h, C.byref(v)))
        return v.value

    def set_trace(self, dev_ptr):
        """Diagnostics: record the launch timeline of the 2-D step into a device u64 buffer
        (mrab_set_trace; dev_ptr 0 turns it off)."""
        _check(lib().mrab_set_trace(self.h, C.c_void_p(int(dev_ptr)) if dev_ptr else None))

    def time_kernel(self, kernel, g, reps=20, flush_l2=True):
        """(ms per launch, algorithmic bytes per launch) of kernel 0 = fused RHS+SAT+AB,
        1 = viscous-flux pass, 2 = donor gather, for mesh g (mrab_time_kernel)."""
        ms, by = C.c_double(), C.c_double()
        _check(lib().mrab_time_kernel(self.h, int(kernel), int(g), int(reps), int(flush_l2),
                                      C.byref(ms), C.byref(by)))
        return ms.value, by.value
