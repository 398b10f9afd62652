"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU checkers.

* ``Oracle``     — the plain-C restatement (liboracle.so, dg2d_oracle.c).
* ``RefSolver``  — the unmodified reference solver compiled from its own sources
                   (_ref/libdg2dref.so via ref_shim.cpp), when it was built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1601_07944_b200 import _lib as L

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdg2dref.so")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)


def _d(a):
    return a.ctypes.data_as(dp)


class OrProblem(C.Structure):
    _fields_ = [("mesh", C.POINTER(L.MeshView)), ("tables", C.POINTER(L.TablesView)),
                ("bc", C.POINTER(L.BcView)), ("gamma", C.c_double), ("flux", C.c_int)]


class OrFail(C.Structure):
    _fields_ = [("pass_", C.c_int), ("id", C.c_int64), ("point", C.c_int), ("rho", C.c_double),
                ("p", C.c_double)]


_olib = None


def oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle liboracle.so`")
        lib = C.CDLL(ORACLE_SO)
        P = C.POINTER(OrProblem)
        F = C.POINTER(OrFail)
        for name, args in {
            "or_volume": [P, dp, dp, F], "or_surface": [P, dp, C.c_double, dp, dp, F],
            "or_rhs": [P, dp, C.c_double, dp, F], "or_limit": [P, dp],
            "or_stable_dt": [P, dp, C.c_double, dp, F],
            "or_step": [P, dp, dp, C.c_double, C.c_int, C.c_int, dp, F],
            "or_run_fixed_steps": [P, dp, dp, C.c_int64, C.c_int, C.c_double, C.c_int, dp, dp, F],
        }.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = C.c_int
        lib.or_gather.argtypes = [P, dp, dp, dp, dp]
        lib.or_gather.restype = None
        lib.or_pressure.argtypes = [dp, C.c_double]
        lib.or_pressure.restype = C.c_double
        lib.or_euler_flux.argtypes = [dp, C.c_double, dp, dp]
        lib.or_euler_flux.restype = None
        lib.or_llf.argtypes = [dp, dp, C.c_double, C.c_double, C.c_double, dp]
        lib.or_llf.restype = None
        lib.or_roe.argtypes = [dp, dp, C.c_double, C.c_double, C.c_double, dp]
        lib.or_roe.restype = None
        lib.or_wave_speed.argtypes = [dp, C.c_double, C.c_double, C.c_double]
        lib.or_wave_speed.restype = C.c_double
        _olib = lib
    return _olib


def bc_view(bc, mesh, tables, keep):
    """Build a dgb_bc_view from a dg2d.BoundaryConditions (same tables the GPU gets)."""
    from paper_1601_07944_b200 import dg2d
    v = L.BcView()
    for m in range(4):
        v.inflow_state[m] = float(bc.inflow_state[m])
    ctx = dg2d.SolverContext.__new__(dg2d.SolverContext)
    ctx.mesh, ctx.tables, ctx.bc = mesh, tables, bc
    dirichlet, wall = dg2d.SolverContext._bc_tables(ctx, 0.0)
    if dirichlet is not None:
        dirichlet = np.ascontiguousarray(dirichlet)
        keep.append(dirichlet)
        v.dirichlet_state = _d(dirichlet)
    if wall is not None:
        wall = np.ascontiguousarray(wall)
        keep.append(wall)
        v.wall_normal = _d(wall)
    if bc.shock is not None:
        s = bc.shock
        v.has_shock = 1
        v.shock_x0, v.shock_angle_deg, v.shock_speed = s.x0, s.angle_deg, s.speed
        for m in range(4):
            v.shock_post[m] = float(s.post[m])
            v.shock_pre[m] = float(s.pre[m])
    return v


class OracleError(RuntimeError):
    pass


class Oracle:
    """The CPU restatement on the same mesh / tables / boundary data as the GPU."""

    def __init__(self, mesh, tables, bc=None, gamma=1.4, flux="llf"):
        from paper_1601_07944_b200 import dg2d
        self.mesh, self.tables = mesh, tables
        self.bc = bc or dg2d.BoundaryConditions()
        self._keep = []
        self._bcv = bc_view(self.bc, mesh, tables, self._keep)
        self.prob = OrProblem(C.pointer(mesh.view), C.pointer(tables.view), C.pointer(self._bcv), gamma,
                              1 if flux == "roe" else 0)
        self.lib = oracle_lib()
        self.shape = (4, tables.n_p, mesh.n_elements())

    def _chk(self, rc, f):
        if rc:
            raise OracleError(f"oracle failure pass={f.pass_} id={f.id} point={f.point} rc={rc}")

    def volume(self, c):
        c = np.ascontiguousarray(c)
        out = np.zeros(self.shape)
        f = OrFail()
        self._chk(self.lib.or_volume(C.byref(self.prob), _d(c), _d(out), C.byref(f)), f)
        return out

    def surface(self, c, t=0.0):
        c = np.ascontiguousarray(c)
        sl = np.zeros((3,) + self.shape)
        sr = np.zeros((3,) + self.shape)
        f = OrFail()
        self._chk(self.lib.or_surface(C.byref(self.prob), _d(c), t, _d(sl), _d(sr), C.byref(f)), f)
        return sl, sr

    def gather(self, vol, sl, sr):
        out = np.zeros(self.shape)
        self.lib.or_gather(C.byref(self.prob), _d(np.ascontiguousarray(vol)), _d(np.ascontiguousarray(sl)),
                           _d(np.ascontiguousarray(sr)), _d(out))
        return out

    def rhs(self, c, t=0.0):
        c = np.ascontiguousarray(c)
        out = np.zeros(self.shape)
        f = OrFail()
        self._chk(self.lib.or_rhs(C.byref(self.prob), _d(c), t, _d(out), C.byref(f)), f)
        return out

    def term_scale(self, c, t=0.0):
        """Per-equation max of (|vol| + sum_q |slot_q|) / detJ (the per-RHS parity scale)."""
        out = np.zeros(4)
        _rchk(self.lib.ref_term_scale(self.h, _d(np.ascontiguousarray(c)), t, _d(out)))
        return out

    def limit(self, c):
        c = np.array(c, np.float64, order="C")
        if self.lib.or_limit(C.byref(self.prob), _d(c)):
            raise ValueError("slope limiting is only supported for p = 1")
        return c

    def stable_dt(self, c, cfl):
        c = np.ascontiguousarray(c)
        dt = C.c_double()
        f = OrFail()
        self._chk(self.lib.or_stable_dt(C.byref(self.prob), _d(c), cfl, C.byref(dt), C.byref(f)), f)
        return dt.value

    def step(self, c, t, dt, scheme, limiting=False):
        c = np.array(c, np.float64, order="C")
        tt = C.c_double(t)
        res = C.c_double()
        f = OrFail()
        self._chk(self.lib.or_step(C.byref(self.prob), _d(c), C.byref(tt), dt, scheme, int(limiting),
                                   C.byref(res), C.byref(f)), f)
        return c, tt.value, res.value

    def run_fixed_steps(self, c, t, n, scheme, cfl, limiting=False):
        c = np.array(c, np.float64, order="C")
        tt = C.c_double(t)
        res = C.c_double()
        hist = np.zeros(max(n, 1))
        f = OrFail()
        self._chk(self.lib.or_run_fixed_steps(C.byref(self.prob), _d(c), C.byref(tt), n, scheme, cfl,
                                              int(limiting), C.byref(res), _d(hist), C.byref(f)), f)
        return c, tt.value, res.value, hist[:n]


# ----------------------------------------------------------------------------- real reference
_rlib = None


def ref_available() -> bool:
    from . import refarm
    return refarm.available()


def ref_lib():
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise ImportError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        from . import refarm
        lib = refarm.lib()  # the -march=native build on the build host's CPU model, else x86-64-v3
        V = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []), "ref_num_threads": (C.c_int, []),
            "ref_mesh_from_msh": (V, [C.c_char_p]),
            "ref_mesh_generate": (V, [C.c_int, C.c_int, C.c_int, dp, C.c_int]),
            "ref_mesh_text": (C.c_int, [C.c_int, C.c_int, C.c_int, dp, C.c_int, C.c_char_p, C.c_size_t,
                                        C.POINTER(C.c_size_t)]),
            "ref_mesh_from_arrays": (V, [C.c_int, dp, dp, C.c_int, ip, ip, dp, dp, dp, C.c_int, C.c_int,
                                         ip, ip, ip, ip, ip, ip, dp, dp, dp]),
            "ref_mesh_free": (None, [V]), "ref_mesh_sizes": (None, [V, ip, ip, ip, ip]),
            "ref_mesh_export": (None, [V, dp, dp, ip, ip, dp, dp, dp, ip, ip, ip, ip, ip, ip, dp, dp, dp]),
            "ref_mesh_dump_edges": (C.c_int, [V, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
            "ref_tables": (V, [C.c_int]), "ref_tables_free": (None, [V]),
            "ref_tables_sizes": (None, [V, ip]),
            "ref_tables_export": (None, [V, dp, dp, dp, dp, dp, dp, dp, dp, dp]),
            "ref_bc_new": (V, []), "ref_bc_free": (None, [V]), "ref_bc_set_inflow": (None, [V, dp]),
            "ref_bc_set_const_dirichlet": (None, [V, dp]), "ref_bc_set_radial_wall": (None, [V]),
            "ref_bc_set_vortex": (None, [V] + [C.c_double] * 6),
            "ref_bc_set_double_mach": (None, [V] + [C.c_double] * 4),
            "ref_bc_set_shock": (None, [V, C.c_double, C.c_double, C.c_double, dp, dp]),
            "ref_bc_eval": (C.c_int, [V, C.c_int, dp, C.c_int, C.c_double, dp]),
            "ref_ctx_new": (V, [V, V, V, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int]),
            "ref_ctx_free": (None, [V]), "ref_ctx_set": (None, [V, C.c_int, C.c_double, C.c_int, C.c_int]),
            "ref_volume": (C.c_int, [V, dp, dp]), "ref_surface": (C.c_int, [V, dp, C.c_double, dp, dp]),
            "ref_gather": (C.c_int, [V, dp, dp, dp, dp]),
            "ref_compute_rhs": (C.c_int, [V, dp, C.c_double, dp]),
            "ref_serial_rhs": (C.c_int, [V, dp, C.c_double, dp]),
            "ref_limit": (C.c_int, [V, dp]), "ref_stable_dt": (C.c_int, [V, dp, dp]),
            "ref_rk_step": (C.c_int, [V, dp, dp, i64p, C.c_double, dp]),
            "ref_run_fixed_steps": (C.c_int, [V, dp, dp, i64p, C.c_int64, dp, dp]),
            "ref_run_to_time": (C.c_int, [V, dp, dp, i64p, C.c_double, C.c_int64, dp]),
            "ref_run_to_steady": (C.c_int, [V, dp, dp, i64p, C.c_double, C.c_int64, i64p, dp, ip, dp,
                                            C.c_int64]),
            "ref_ssp_step": (C.c_int, [V, dp, dp, i64p, C.c_double, C.c_int, C.c_int, dp]),
            "ref_total_mass": (C.c_double, [V, dp]),
            "ref_project": (C.c_int, [V, V, C.c_double, C.c_int, dp, dp]),
            "ref_mesh_periodic_box": (V, [C.c_int, C.c_int, C.c_double, C.c_double]),
            "ref_term_scale": (C.c_int, [V, dp, C.c_double, dp]),
            "ref_project_isentropic_vortex": (C.c_int, [V, V] + [C.c_double] * 8 + [dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _rlib = lib
    return _rlib


class RefError(RuntimeError):
    pass


def _rchk(rc):
    if rc:
        raise RefError(f"[{rc}] " + ref_lib().ref_last_error().decode())


class RefMesh:
    def __init__(self, handle):
        if not handle:
            raise RefError(ref_lib().ref_last_error().decode())
        self.h = handle
        lib = ref_lib()
        nv, ne, ned, nb = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib.ref_mesh_sizes(handle, C.byref(nv), C.byref(ne), C.byref(ned), C.byref(nb))
        self.nv, self.ne, self.ned, self.nb = nv.value, ne.value, ned.value, nb.value

    @classmethod
    def generate(cls, kind, nx, ny, *params):
        p = (C.c_double * max(1, len(params)))(*params)
        return cls(ref_lib().ref_mesh_generate(kind, nx, ny, p, len(params)))

    @classmethod
    def from_msh(cls, text):
        return cls(ref_lib().ref_mesh_from_msh(text.encode()))

    @classmethod
    def from_mesh(cls, m):
        """Reference Mesh holding exactly our mesh arrays (for sizes beyond the text path)."""
        lib = ref_lib()
        a = dict(vx=m.vx, vy=m.vy, ev=np.ascontiguousarray(m.elem_v), ee=np.ascontiguousarray(m.elem_edge),
                 det=m.det_jac, tau=np.ascontiguousarray(m.tau), inr=m.inradius)
        ip_ = lambda x: np.ascontiguousarray(x, np.int32).ctypes.data_as(ip)
        keep = [np.ascontiguousarray(x) for x in a.values()]
        h = lib.ref_mesh_from_arrays(
            len(m.vx), _d(keep[0]), _d(keep[1]), m.n_elements(), ip_(keep[2]), ip_(keep[3]),
            _d(keep[4]), _d(keep[5]), _d(keep[6]), m.n_edges(), m.n_boundary_edges,
            ip_(m.edge_v0), ip_(m.edge_v1), ip_(m.edge_left), ip_(m.edge_right),
            ip_(m.edge_side_left), ip_(m.edge_side_right),
            _d(m.edge_nx), _d(m.edge_ny), _d(m.edge_half_length))
        return cls(h)

    def export(self):
        out = dict(vx=np.zeros(self.nv), vy=np.zeros(self.nv), elem_v=np.zeros((self.ne, 3), np.int32),
                   elem_edge=np.zeros((self.ne, 3), np.int32), det_jac=np.zeros(self.ne),
                   tau=np.zeros((self.ne, 4)), inradius=np.zeros(self.ne),
                   edge_v0=np.zeros(self.ned, np.int32), edge_v1=np.zeros(self.ned, np.int32),
                   edge_left=np.zeros(self.ned, np.int32), edge_right=np.zeros(self.ned, np.int32),
                   edge_side_left=np.zeros(self.ned, np.int32), edge_side_right=np.zeros(self.ned, np.int32),
                   edge_nx=np.zeros(self.ned), edge_ny=np.zeros(self.ned), edge_half_length=np.zeros(self.ned))
        o = out
        ptr = lambda x: x.ctypes.data_as(ip) if x.dtype == np.int32 else _d(x)
        ref_lib().ref_mesh_export(self.h, *[ptr(o[k]) for k in (
            "vx", "vy", "elem_v", "elem_edge", "det_jac", "tau", "inradius", "edge_v0", "edge_v1",
            "edge_left", "edge_right", "edge_side_left", "edge_side_right", "edge_nx", "edge_ny",
            "edge_half_length")])
        return out

    def dump_edges(self):
        need = C.c_size_t()
        ref_lib().ref_mesh_dump_edges(self.h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        ref_lib().ref_mesh_dump_edges(self.h, buf, need.value, C.byref(need))
        return buf.value.decode()

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_mesh_free(self.h)
            self.h = None


class RefTables:
    def __init__(self, p):
        lib = ref_lib()
        self.h = lib.ref_tables(p)
        if not self.h:
            raise RefError(lib.ref_last_error().decode())
        s = (C.c_int * 5)()
        lib.ref_tables_sizes(self.h, s)
        self.p, self.n_p, self.n_quad, self.n_edge_pts, self.total_stored_doubles = list(s)
        nq, np_, k = self.n_quad, self.n_p, self.n_edge_pts
        self.phi_interior = np.zeros((nq, np_))
        self.dphi_dr_interior = np.zeros((nq, np_))
        self.dphi_ds_interior = np.zeros((nq, np_))
        self.w_interior = np.zeros(nq)
        self.r_interior = np.zeros((nq, 2))
        self.phi_edge = np.zeros((3, k, np_))
        self.w_edge = np.zeros(k)
        self.xi_edge = np.zeros(k)
        self.phi_edge_mid = np.zeros((3, np_))
        lib.ref_tables_export(self.h, _d(self.phi_interior), _d(self.dphi_dr_interior),
                              _d(self.dphi_ds_interior), _d(self.w_interior), _d(self.r_interior),
                              _d(self.phi_edge), _d(self.w_edge), _d(self.xi_edge), _d(self.phi_edge_mid))

    def as_external(self):
        from paper_1601_07944_b200 import dg2d
        return dg2d.ExternalTables(self.p, self.phi_interior, self.dphi_dr_interior, self.dphi_ds_interior,
                                   self.w_interior, self.r_interior, self.phi_edge, self.w_edge,
                                   self.xi_edge, self.phi_edge_mid)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_tables_free(self.h)
            self.h = None


class RefBC:
    def __init__(self):
        self.h = ref_lib().ref_bc_new()

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_bc_free(self.h)
            self.h = None


class RefSolver:
    """The reference's SolverContext + passes on a RefMesh / RefTables / RefBC."""

    def __init__(self, mesh: RefMesh, tables: RefTables, bc: RefBC = None, gamma=1.4, rk_order=4, cfl=0.3,
                 limiting=False, workers=0):
        self.mesh, self.tables = mesh, tables
        self.bc = bc or RefBC()
        self.lib = ref_lib()
        self.h = self.lib.ref_ctx_new(mesh.h, tables.h, self.bc.h, gamma, rk_order, cfl, int(limiting), workers)
        self.shape = (4, tables.n_p, mesh.ne)

    def set(self, rk_order=4, cfl=0.3, limiting=False, workers=0):
        self.lib.ref_ctx_set(self.h, rk_order, cfl, int(limiting), workers)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_ctx_free(self.h)
            self.h = None

    def volume(self, c):
        out = np.zeros(self.shape)
        _rchk(self.lib.ref_volume(self.h, _d(np.ascontiguousarray(c)), _d(out)))
        return out

    def surface(self, c, t=0.0):
        sl = np.zeros((3,) + self.shape)
        sr = np.zeros((3,) + self.shape)
        _rchk(self.lib.ref_surface(self.h, _d(np.ascontiguousarray(c)), t, _d(sl), _d(sr)))
        return sl, sr

    def gather(self, vol, sl, sr):
        out = np.zeros(self.shape)
        _rchk(self.lib.ref_gather(self.h, _d(np.ascontiguousarray(vol)), _d(np.ascontiguousarray(sl)),
                                  _d(np.ascontiguousarray(sr)), _d(out)))
        return out

    def rhs(self, c, t=0.0):
        out = np.zeros(self.shape)
        _rchk(self.lib.ref_compute_rhs(self.h, _d(np.ascontiguousarray(c)), t, _d(out)))
        return out

    def serial_rhs(self, c, t=0.0):
        out = np.zeros(self.shape)
        _rchk(self.lib.ref_serial_rhs(self.h, _d(np.ascontiguousarray(c)), t, _d(out)))
        return out

    def term_scale(self, c, t=0.0):
        """Per-equation max of (|vol| + sum_q |slot_q|) / detJ (the per-RHS parity scale)."""
        out = np.zeros(4)
        _rchk(self.lib.ref_term_scale(self.h, _d(np.ascontiguousarray(c)), t, _d(out)))
        return out

    def limit(self, c):
        c = np.array(c, np.float64, order="C")
        _rchk(self.lib.ref_limit(self.h, _d(c)))
        return c

    def stable_dt(self, c):
        dt = C.c_double()
        _rchk(self.lib.ref_stable_dt(self.h, _d(np.ascontiguousarray(c)), C.byref(dt)))
        return dt.value

    def rk_step(self, c, t, dt, step=0):
        c = np.array(c, np.float64, order="C")
        tt, ss, res = C.c_double(t), C.c_int64(step), C.c_double()
        _rchk(self.lib.ref_rk_step(self.h, _d(c), C.byref(tt), C.byref(ss), dt, C.byref(res)))
        return c, tt.value, res.value

    def ssp_step(self, c, t, dt, scheme, limiting=False, step=0):
        c = np.array(c, np.float64, order="C")
        tt, ss, res = C.c_double(t), C.c_int64(step), C.c_double()
        _rchk(self.lib.ref_ssp_step(self.h, _d(c), C.byref(tt), C.byref(ss), dt, scheme, int(limiting),
                                    C.byref(res)))
        return c, tt.value, res.value

    def run_fixed_steps(self, c, t, n, step=0):
        c = np.array(c, np.float64, order="C")
        tt, ss, res = C.c_double(t), C.c_int64(step), C.c_double()
        hist = np.zeros(max(n, 1))
        rc = self.lib.ref_run_fixed_steps(self.h, _d(c), C.byref(tt), C.byref(ss), n, C.byref(res), _d(hist))
        _rchk(rc)
        return c, tt.value, res.value, hist[:n]

    def run_to_time(self, c, t, t_end, max_steps, step=0):
        c = np.array(c, np.float64, order="C")
        tt, ss, res = C.c_double(t), C.c_int64(step), C.c_double()
        _rchk(self.lib.ref_run_to_time(self.h, _d(c), C.byref(tt), C.byref(ss), t_end, max_steps, C.byref(res)))
        return c, tt.value, ss.value, res.value

    def run_to_steady(self, c, tol, max_steps, t=0.0, step=0):
        c = np.array(c, np.float64, order="C")
        tt, ss, steps, res, conv = C.c_double(t), C.c_int64(step), C.c_int64(), C.c_double(), C.c_int()
        cap = int(min(max_steps, 1 << 20))
        hist = np.zeros(max(cap, 1))
        _rchk(self.lib.ref_run_to_steady(self.h, _d(c), C.byref(tt), C.byref(ss), tol, max_steps,
                                         C.byref(steps), C.byref(res), C.byref(conv), _d(hist), cap))
        return c, steps.value, res.value, bool(conv.value), hist[:min(steps.value, cap)]

    def total_mass(self, c):
        return self.lib.ref_total_mass(self.h, _d(np.ascontiguousarray(c)))


def ref_export(mesh: "RefMesh", tables: "RefTables", coeffs, path, csv=False, gamma=1.4):
    """The reference's export_vtk / export_csv (output.cpp:30-81) on the same coefficients."""
    lib = ref_lib()
    lib.ref_export.argtypes = [C.c_void_p, C.c_void_p, C.c_double, dp, C.c_int, C.c_char_p]
    c = np.ascontiguousarray(coeffs, np.float64)
    _rchk(lib.ref_export(mesh.h, tables.h, gamma, _d(c), int(csv), path.encode()))


def ref_project(mesh: RefMesh, tables: RefTables, kind, params, gamma=1.4):
    out = np.zeros((4, tables.n_p, mesh.ne))
    p = (C.c_double * max(1, len(params)))(*params)
    _rchk(ref_lib().ref_project(mesh.h, tables.h, gamma, kind, p, _d(out)))
    return out
