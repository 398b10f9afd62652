"""Python mirror of the reference solver interface, backed by the B200 kernels.

Names, argument meaning and error behaviour follow the reference's C++ API
(``/root/reference/proj/include/dg2d/*.hpp``) so that the parity tests read like
the reference's own tests:

* ``Mesh`` / ``parse_msh`` / ``build_connectivity`` / ``gen_*_msh`` (mesh.hpp, problems.hpp)
* ``build_tables`` / ``eval_basis`` (basis.hpp)
* ``BoundaryConditions`` / ``MovingShock`` / ``vortex_boundary`` / ``double_mach_boundary`` (euler.hpp, problems.hpp)
* ``SolverContext`` / ``SolverOptions`` / ``SolverState`` / ``RhsBuffers`` (solver.hpp:46-95)
* ``project_initial``, ``eval_volume_pass``, ``eval_surface_pass``, ``eval_rhs_pass``,
  ``compute_rhs``, ``limit``, ``stable_dt``, ``rk_step``, ``run_to_steady``,
  ``run_to_time``, ``run_fixed_steps``, ``save_checkpoint``, ``load_checkpoint``,
  ``total_mass``, ``max_abs_diff`` (solver.hpp:98-155)

Coefficient arrays are numpy float64 arrays of shape (4, n_p, n_elem), i.e.
exactly the reference's ``CoefficientArray::data`` layout.  Every solver call
runs on the GPU through the C ABI; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
import struct
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from ._lib import dptr, iptr, lib

kEq = 4
kMaxDegree = 5


# ----------------------------------------------------------------------------- errors
class SolverAbort(RuntimeError):
    """solver.hpp:14-16"""


class MeshError(RuntimeError):
    """mesh.hpp:15-17"""


class ConfigError(RuntimeError):
    """config.hpp:11-13"""


def _check(rc: int):
    if rc == L.OK:
        return
    msg = L.last_message()
    if rc in (L.ERR_INADMISSIBLE, L.ERR_BC, L.ERR_NOT_REACHED):
        raise SolverAbort(msg)
    if rc == L.ERR_MESH:
        raise MeshError(msg)
    if rc == L.ERR_ARG:
        raise ValueError(msg)  # std::invalid_argument
    if rc == L.ERR_IO:
        raise OSError(msg)
    raise RuntimeError(msg)


def basis_count(p: int) -> int:
    return (p + 1) * (p + 2) // 2


@dataclasses.dataclass
class GasModel:
    gamma: float = 1.4


# ----------------------------------------------------------------------------- mesh
class MeshPrecursor:
    """Raw mesh-file content before connectivity (mesh.hpp:66-77); kept as text."""

    def __init__(self, text: str):
        self.text = text


def parse_msh(text: str) -> MeshPrecursor:
    return MeshPrecursor(text)


def parse_msh_file(path: str) -> MeshPrecursor:
    try:
        with open(path, "r") as f:
            return MeshPrecursor(f.read())
    except OSError:
        raise MeshError(f"cannot open mesh file '{path}'")


class Mesh:
    """Connectivity-complete mesh (mesh.hpp:46-63), SoA numpy views."""

    def __init__(self, handle):
        self._h = handle
        v = L.MeshView()
        _check(lib.dgb_mesh_get_view(handle, C.byref(v)))
        self._view = v
        n, ne, nv = v.n_elements, v.n_edges, v.n_vertices

        def arr(ptr, count, dtype):
            if count == 0:
                return np.zeros(0, dtype)
            return np.ctypeslib.as_array(ptr, shape=(count,)).view(dtype)

        self.vx = arr(v.vx, nv, np.float64)
        self.vy = arr(v.vy, nv, np.float64)
        self.elem_v = arr(v.elem_v, 3 * n, np.int32).reshape(n, 3)
        self.elem_edge = arr(v.elem_edge, 3 * n, np.int32).reshape(n, 3)
        self.det_jac = arr(v.det_jac, n, np.float64)
        self.tau = arr(v.tau, 4 * n, np.float64).reshape(n, 4)
        self.inradius = arr(v.inradius, n, np.float64)
        self.edge_v0 = arr(v.edge_v0, ne, np.int32)
        self.edge_v1 = arr(v.edge_v1, ne, np.int32)
        self.edge_left = arr(v.edge_left, ne, np.int32)
        self.edge_right = arr(v.edge_right, ne, np.int32)
        self.edge_side_left = arr(v.edge_side_left, ne, np.int32)
        self.edge_side_right = arr(v.edge_side_right, ne, np.int32)
        self.edge_nx = arr(v.edge_nx, ne, np.float64)
        self.edge_ny = arr(v.edge_ny, ne, np.float64)
        self.edge_half_length = arr(v.edge_half_length, ne, np.float64)
        self.n_boundary_edges = v.n_boundary_edges

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.dgb_mesh_free(h)
            self._h = None

    @property
    def view(self) -> L.MeshView:
        return self._view

    def n_elements(self) -> int:
        return self._view.n_elements

    def n_edges(self) -> int:
        return self._view.n_edges

    def neighbor(self, i: int, q: int) -> int:
        e = self.elem_edge[i, q]
        return int(self.edge_right[e] if self.edge_left[e] == i else self.edge_left[e])

    def total_area(self) -> float:
        return float(np.sum(0.5 * self.det_jac))

    def vertex_of(self, elem: int, local: int):
        v = self.elem_v[elem, local]
        return float(self.vx[v]), float(self.vy[v])

    def dump_edges(self) -> str:
        need = C.c_size_t()
        _check(lib.dgb_mesh_dump_edges(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(lib.dgb_mesh_dump_edges(self._h, buf, need.value, C.byref(need)))
        return buf.value.decode()


class ArrayMesh(Mesh):
    """A mesh given as arrays (e.g. a reference ``Mesh`` exported field by field)."""

    _FIELDS = ("vx", "vy", "elem_v", "elem_edge", "det_jac", "tau", "inradius", "edge_v0", "edge_v1",
               "edge_left", "edge_right", "edge_side_left", "edge_side_right", "edge_nx", "edge_ny",
               "edge_half_length")

    def __init__(self, arrays: dict, n_boundary_edges: Optional[int] = None):
        self._h = None
        for k in self._FIELDS:
            a = np.asarray(arrays[k])
            dt = np.int32 if a.dtype.kind in "iu" else np.float64
            setattr(self, k, np.ascontiguousarray(a, dt))
        n, ne = self.det_jac.shape[0], self.edge_v0.shape[0]
        self.elem_v = self.elem_v.reshape(n, 3)
        self.elem_edge = self.elem_edge.reshape(n, 3)
        self.tau = self.tau.reshape(n, 4)
        if n_boundary_edges is None:
            n_boundary_edges = int(np.count_nonzero(self.edge_right < 0))
        self.n_boundary_edges = n_boundary_edges
        v = L.MeshView()
        v.n_vertices, v.vx, v.vy = self.vx.shape[0], dptr(self.vx), dptr(self.vy)
        v.n_elements, v.elem_v, v.elem_edge = n, iptr(self.elem_v), iptr(self.elem_edge)
        v.det_jac, v.tau, v.inradius = dptr(self.det_jac), dptr(self.tau), dptr(self.inradius)
        v.n_edges, v.n_boundary_edges = ne, n_boundary_edges
        v.edge_v0, v.edge_v1 = iptr(self.edge_v0), iptr(self.edge_v1)
        v.edge_left, v.edge_right = iptr(self.edge_left), iptr(self.edge_right)
        v.edge_side_left, v.edge_side_right = iptr(self.edge_side_left), iptr(self.edge_side_right)
        v.edge_nx, v.edge_ny, v.edge_half_length = dptr(self.edge_nx), dptr(self.edge_ny), dptr(self.edge_half_length)
        self._view = v

    def dump_edges(self) -> str:
        rows = []
        for k in range(self.edge_v0.shape[0]):
            rows.append("%d %d %d %d %d %d %.17g %.17g %.17g\n" % (
                self.edge_v0[k], self.edge_v1[k], self.edge_left[k], self.edge_right[k], self.edge_side_left[k],
                self.edge_side_right[k], self.edge_nx[k], self.edge_ny[k], self.edge_half_length[k]))
        return "".join(rows)


def build_connectivity(pre: MeshPrecursor) -> Mesh:
    h = C.c_void_p()
    raw = pre.text.encode()
    _check(lib.dgb_mesh_from_msh(raw, len(raw), C.byref(h)))
    return Mesh(h)


def _params(vals):
    a = (C.c_double * max(1, len(vals)))(*vals)
    return a, len(vals)


def generate_mesh(kind: int, nx: int, ny: int, *params) -> Mesh:
    """Direct structured generator, bit-identical to build_connectivity(parse_msh(gen_*_msh(..)))."""
    h = C.c_void_p()
    p, n = _params(params)
    _check(lib.dgb_mesh_generate(kind, nx, ny, p, n, C.byref(h)))
    return Mesh(h)


def _gen_text(kind, nx, ny, *params) -> str:
    p, n = _params(params)
    need = C.c_size_t()
    _check(lib.dgb_mesh_generate_text(kind, nx, ny, p, n, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(lib.dgb_mesh_generate_text(kind, nx, ny, p, n, buf, need.value, C.byref(need)))
    return buf.value.decode()


def gen_box_msh(nx, ny, width, height, tag) -> str:
    return _gen_text(L.MESH_BOX, nx, ny, width, height, tag)


def gen_sheared_box_msh(nx, ny, width, height, shear, tag) -> str:
    return _gen_text(L.MESH_SHEARED_BOX, nx, ny, width, height, shear, tag)


def gen_double_mach_msh(nx, ny, x0=1.0 / 6.0) -> str:
    return _gen_text(L.MESH_DOUBLE_MACH, nx, ny, x0)


@dataclasses.dataclass
class VortexGeometry:
    """problems.hpp:14-20"""
    r_inner: float = 1.0
    r_outer: float = 1.384
    mach_inner: float = 2.25
    rho_inner: float = 1.0
    sound_speed_inner: float = 1.0


def gen_vortex_msh(level, geo: VortexGeometry = VortexGeometry()) -> str:
    if level < 0 or level > 5:
        raise ValueError("vortex mesh level must be 0..5")
    return _gen_text(L.MESH_VORTEX, level, 0, geo.r_inner, geo.r_outer)


def two_triangle_square(tag=1) -> str:
    return gen_box_msh(1, 1, 1.0, 1.0, tag)


# ----------------------------------------------------------------------------- tables
class BasisTables:
    """basis.hpp:48-82"""

    def __init__(self, p: int):
        h = C.c_void_p()
        _check(lib.dgb_tables_build(p, C.byref(h)))
        self._h = h
        v = L.TablesView()
        _check(lib.dgb_tables_get_view(h, C.byref(v)))
        self._view = v
        self.p, self.n_p, self.n_quad, self.n_edge_pts = v.p, v.n_p, v.n_quad, v.n_edge_pts
        nq, np_, k = v.n_quad, v.n_p, v.n_edge_pts

        def arr(ptr, count):
            return np.ctypeslib.as_array(ptr, shape=(count,))

        self.phi_interior = arr(v.phi_interior, nq * np_).reshape(nq, np_)
        self.dphi_dr_interior = arr(v.dphi_dr_interior, nq * np_).reshape(nq, np_)
        self.dphi_ds_interior = arr(v.dphi_ds_interior, nq * np_).reshape(nq, np_)
        self.w_interior = arr(v.w_interior, nq)
        self.r_interior = arr(v.r_interior, 2 * nq).reshape(nq, 2)
        self.phi_edge = arr(v.phi_edge, 3 * k * np_).reshape(3, k, np_)
        self.w_edge = arr(v.w_edge, k)
        self.xi_edge = arr(v.xi_edge, k)
        self.phi_edge_mid = arr(v.phi_edge_mid, 3 * np_).reshape(3, np_)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.dgb_tables_free(h)
            self._h = None

    @property
    def view(self) -> L.TablesView:
        return self._view

    def phi_side(self, q, k, j):
        return float(self.phi_edge[q - 1, k, j])


class ExternalTables:
    """Tables supplied as arrays (e.g. the reference's own build_tables output)."""

    def __init__(self, p, phi, dr, ds, w, rs, phe, we, xi, phm):
        self.p = p
        self.n_p = phi.shape[1]
        self.n_quad = phi.shape[0]
        self.n_edge_pts = we.shape[0]
        self.phi_interior = np.ascontiguousarray(phi, np.float64)
        self.dphi_dr_interior = np.ascontiguousarray(dr, np.float64)
        self.dphi_ds_interior = np.ascontiguousarray(ds, np.float64)
        self.w_interior = np.ascontiguousarray(w, np.float64)
        self.r_interior = np.ascontiguousarray(rs, np.float64).reshape(-1, 2)
        self.phi_edge = np.ascontiguousarray(phe, np.float64).reshape(3, self.n_edge_pts, self.n_p)
        self.w_edge = np.ascontiguousarray(we, np.float64)
        self.xi_edge = np.ascontiguousarray(xi, np.float64)
        self.phi_edge_mid = np.ascontiguousarray(phm, np.float64).reshape(3, self.n_p)
        v = L.TablesView()
        v.p, v.n_p, v.n_quad, v.n_edge_pts = p, self.n_p, self.n_quad, self.n_edge_pts
        v.phi_interior = dptr(self.phi_interior)
        v.dphi_dr_interior = dptr(self.dphi_dr_interior)
        v.dphi_ds_interior = dptr(self.dphi_ds_interior)
        v.w_interior = dptr(self.w_interior)
        v.r_interior = dptr(self.r_interior)
        v.phi_edge = dptr(self.phi_edge)
        v.w_edge = dptr(self.w_edge)
        v.xi_edge = dptr(self.xi_edge)
        v.phi_edge_mid = dptr(self.phi_edge_mid)
        self._view = v

    @property
    def view(self):
        return self._view


def build_tables(p: int) -> BasisTables:
    return BasisTables(p)


def eval_basis(p, j, rs):
    phi = C.c_double()
    _check(lib.dgb_eval_basis(p, j, rs[0], rs[1], C.byref(phi), None, None))
    return phi.value


def eval_basis_grad(p, j, rs):
    dr, ds = C.c_double(), C.c_double()
    _check(lib.dgb_eval_basis(p, j, rs[0], rs[1], None, C.byref(dr), C.byref(ds)))
    return dr.value, ds.value


# ----------------------------------------------------------------------------- physics helpers
def make_state(rho, u, v, p, gamma=1.4):
    return np.array([rho, rho * u, rho * v, p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)])


def pressure(u, gas: GasModel = GasModel()):
    u = np.asarray(u, np.float64)
    return (gas.gamma - 1.0) * (u[..., 3] - 0.5 * (u[..., 1] ** 2 + u[..., 2] ** 2) / u[..., 0])


def interior_points(mesh: Mesh, tables) -> np.ndarray:
    xy = np.empty((mesh.n_elements(), tables.n_quad, 2))
    _check(lib.dgb_interior_points(C.byref(mesh.view), C.byref(tables.view), dptr(xy)))
    return xy


def boundary_points(mesh: Mesh, tables) -> np.ndarray:
    xy = np.empty((max(mesh.n_boundary_edges, 0), tables.n_edge_pts, 2))
    if mesh.n_boundary_edges:
        _check(lib.dgb_boundary_points(C.byref(mesh.view), C.byref(tables.view), dptr(xy)))
    return xy


def vortex_exact(xy, geo: VortexGeometry = VortexGeometry(), gas: GasModel = GasModel()):
    xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
    out = np.empty((xy.shape[0], 4))
    _check(lib.dgb_vortex_exact(dptr(xy), xy.shape[0], geo.r_inner, geo.r_outer, geo.mach_inner,
                                geo.rho_inner, geo.sound_speed_inner, gas.gamma, dptr(out)))
    return out


def rankine_hugoniot_post(pre, mach, n, gas: GasModel = GasModel()):
    pre = np.ascontiguousarray(pre, np.float64)
    out = np.empty(4)
    _check(lib.dgb_rankine_hugoniot_post(dptr(pre), mach, n[0], n[1], gas.gamma, dptr(out)))
    return out


@dataclasses.dataclass
class IsentropicVortex:
    """Shu's isentropic vortex on a periodic box (BASELINE.json configs; not in the reference)."""
    xc: float = 5.0
    yc: float = 5.0
    beta: float = 5.0
    u_inf: float = 1.0
    v_inf: float = 1.0
    width: float = 10.0
    height: float = 10.0

    def __call__(self, xy, t=0.0, gas: GasModel = GasModel()):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        out = np.empty((xy.shape[0], 4))
        _check(lib.dgb_isentropic_vortex(dptr(xy), xy.shape[0], self.xc, self.yc, self.beta, self.u_inf,
                                         self.v_inf, self.width, self.height, t, gas.gamma, dptr(out)))
        return out


# ----------------------------------------------------------------------------- boundary conditions
@dataclasses.dataclass
class MovingShock:
    """euler.hpp:91-102"""
    x0: float = 0.0
    angle_deg: float = 60.0
    speed: float = 10.0
    post: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(4))
    pre: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(4))


@dataclasses.dataclass
class BoundaryConditions:
    """euler.hpp:104-111.  ``dirichlet(xy[n,2], t) -> states[n,4]`` and
    ``wall_normal(xy[n,2]) -> normals[n,2]`` are vectorised closures; they are
    evaluated once at every boundary Gauss point when the device context is built
    (``time_dependent=True`` re-evaluates the Dirichlet table before each RHS)."""
    inflow_state: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(4))
    dirichlet: Optional[Callable] = None
    wall_normal: Optional[Callable] = None
    shock: Optional[MovingShock] = None
    time_dependent: bool = False


def vortex_boundary(geo: VortexGeometry = VortexGeometry(), gas: GasModel = GasModel()) -> BoundaryConditions:
    """problems.cpp:68-77"""
    inflow = vortex_exact(np.array([[0.5 * (geo.r_inner + geo.r_outer), 0.0]]), geo, gas)[0]
    return BoundaryConditions(
        inflow_state=inflow,
        dirichlet=lambda xy, t: vortex_exact(xy, geo, gas),
        wall_normal=lambda xy: xy / np.hypot(xy[:, 0], xy[:, 1])[:, None])


@dataclasses.dataclass
class DoubleMachSetup:
    """problems.hpp:34-44, problems.cpp:96-100"""
    x0: float = 1.0 / 6.0
    shock_mach: float = 10.0
    angle_deg: float = 60.0
    pre: np.ndarray = dataclasses.field(default_factory=lambda: np.array([1.4, 0.0, 0.0, 1.0 / 0.4]))
    post: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.post is None:
            rad = self.angle_deg * math.pi / 180.0
            self.post = rankine_hugoniot_post(self.pre, self.shock_mach, (math.sin(rad), -math.cos(rad)))


def double_mach_boundary(setup: DoubleMachSetup, gas: GasModel = GasModel()) -> BoundaryConditions:
    """problems.cpp:102-115"""
    p_pre = (1.4 - 1.0) * (setup.pre[3] - 0.5 * (setup.pre[1] ** 2 + setup.pre[2] ** 2) / setup.pre[0])
    c_pre = math.sqrt(1.4 * p_pre / setup.pre[0])
    return BoundaryConditions(
        inflow_state=np.array(setup.post, np.float64),
        shock=MovingShock(setup.x0, setup.angle_deg, setup.shock_mach * c_pre,
                          np.array(setup.post, np.float64), np.array(setup.pre, np.float64)))


def double_mach_initial(xy, setup: DoubleMachSetup):
    """problems.cpp:117-121 (vectorised)"""
    xy = np.asarray(xy).reshape(-1, 2)
    rad = setup.angle_deg * math.pi / 180.0
    front = setup.x0 + xy[:, 1] * math.cos(rad) / math.sin(rad)
    return np.where((xy[:, 0] < front)[:, None], setup.post[None, :], setup.pre[None, :])


# ----------------------------------------------------------------------------- solver
@dataclasses.dataclass
class SolverOptions:
    """solver.hpp:72-78 plus the scheme selector for the SSP schemes (new)."""
    rk_order: int = 4
    cfl: float = 0.3
    limiting: bool = False
    workers: int = 0
    chunk: int = 256
    scheme: Optional[int] = None  # None -> rk_order (2 midpoint / 4 classic); 102 SSP-RK2, 103 SSP-RK3
    flux: str = "llf"  # "llf" (euler.hpp:59-71) or "roe" (new, BASELINE.json north star)

    def scheme_id(self) -> int:
        return self.scheme if self.scheme is not None else self.rk_order

    def flux_id(self) -> int:
        if self.flux not in ("llf", "roe"):
            raise ValueError(f"unknown numerical flux {self.flux!r}")
        return L.FLUX_ROE if self.flux == "roe" else L.FLUX_LLF


@dataclasses.dataclass
class PassTimers:
    volume: float = 0.0
    surface: float = 0.0
    rhs: float = 0.0
    limiter: float = 0.0
    other: float = 0.0
    stage: float = 0.0


@dataclasses.dataclass
class SolverState:
    coeffs: np.ndarray
    t: float = 0.0
    step_count: int = 0


@dataclasses.dataclass
class SteadyResult:
    steps: int = 0
    residual: float = 0.0
    converged: bool = False


class RhsBuffers:
    """solver.hpp:46-62: volume [4][n_p][N], surface_left/right [3][4][n_p][N]."""

    def __init__(self, n_eq, n_modes, n_elem):
        self.volume = np.zeros((n_eq, n_modes, n_elem))
        self.surface_left = np.zeros((3, n_eq, n_modes, n_elem))
        self.surface_right = np.zeros((3, n_eq, n_modes, n_elem))


class SolverContext:
    """solver.hpp:80-87 plus the device context it owns (created lazily)."""

    def __init__(self, mesh: Mesh, tables, gas: GasModel = None, bc: BoundaryConditions = None,
                 options: SolverOptions = None, device: Optional[int] = None):
        self.mesh = mesh
        self.tables = tables
        self.gas = gas or GasModel()
        self.bc = bc or BoundaryConditions()
        self.options = options or SolverOptions()
        self.device = device if device is not None else int(os.environ.get("DG2D_DEVICE", "0"))
        self.timers = PassTimers()
        self._ctx = None
        self._keep = []

    # -- device context -------------------------------------------------------
    def _bc_tables(self, t=0.0):
        mesh, tb, bc = self.mesh, self.tables, self.bc
        nb = mesh.n_boundary_edges
        codes = mesh.edge_right[:nb]
        xy = boundary_points(mesh, tb).reshape(-1, 2)
        dirichlet = wall = None
        if bc.dirichlet is not None and nb:
            mask = np.repeat(codes == -3, tb.n_edge_pts)
            dirichlet = np.zeros((xy.shape[0], 4))
            if mask.any():
                dirichlet[mask] = np.asarray(bc.dirichlet(xy[mask], t), np.float64).reshape(-1, 4)
        if bc.wall_normal is not None and nb:
            mask = np.repeat(codes == -2, tb.n_edge_pts)
            wall = np.zeros((xy.shape[0], 2))
            if mask.any():
                wall[mask] = np.asarray(bc.wall_normal(xy[mask]), np.float64).reshape(-1, 2)
        return dirichlet, wall

    def _bc_view(self):
        """dgb_bc_view of the boundary conditions (arrays kept alive on self)."""
        dirichlet, wall = self._bc_tables(0.0)
        v = L.BcView()
        for m in range(4):
            v.inflow_state[m] = float(self.bc.inflow_state[m])
        if dirichlet is not None:
            dirichlet = np.ascontiguousarray(dirichlet)
            v.dirichlet_state = dptr(dirichlet)
        if wall is not None:
            wall = np.ascontiguousarray(wall)
            v.wall_normal = dptr(wall)
        if self.bc.shock is not None:
            s = self.bc.shock
            v.has_shock = 1
            v.shock_x0, v.shock_angle_deg, v.shock_speed = s.x0, s.angle_deg, s.speed
            for m in range(4):
                v.shock_post[m] = float(s.post[m])
                v.shock_pre[m] = float(s.pre[m])
        self._keep = [dirichlet, wall]
        return v

    @property
    def handle(self):
        if self._ctx is None:
            v = self._bc_view()
            h = C.c_void_p()
            _check(lib.dgb_create(C.byref(self.mesh.view), C.byref(self.tables.view), C.byref(v),
                                  self.gas.gamma, self.device, C.byref(h)))
            self._ctx = h
            lib.dgb_enable_timers(h, 1)
            _check(lib.dgb_set_flux(h, self.options.flux_id()))
        return self._ctx

    def close(self):
        if self._ctx is not None:
            lib.dgb_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _refresh_bc(self, t):
        if self.bc.time_dependent and self.bc.dirichlet is not None:
            dirichlet, _ = self._bc_tables(t)
            if dirichlet is not None:
                dirichlet = np.ascontiguousarray(dirichlet)
                _check(lib.dgb_set_dirichlet(self.handle, dptr(dirichlet)))

    def _shape(self):
        return (kEq, self.tables.n_p, self.mesh.n_elements())

    def upload(self, slot, coeffs):
        c = np.ascontiguousarray(coeffs, np.float64)
        if c.shape != self._shape():
            raise ValueError(f"coefficient array has shape {c.shape}, expected {self._shape()}")
        _check(lib.dgb_upload(self.handle, slot, dptr(c)))

    def download(self, slot):
        out = np.empty(self._shape())
        _check(lib.dgb_download(self.handle, slot, dptr(out)))
        return out

    def read_timers(self):
        t = L.PassTimers()
        _check(lib.dgb_timers(self.handle, C.byref(t)))
        self.timers = PassTimers(t.volume, t.surface, t.rhs, t.limiter, t.other, t.stage)
        return self.timers

    def launch_count(self) -> int:
        return int(lib.dgb_launch_count(self.handle))


def project_initial(u0: Callable, mesh: Mesh, tables, gas: GasModel = GasModel()) -> np.ndarray:
    """solver.cpp:74-97: L2 projection of ``u0(xy[n,2]) -> states[n,4]``."""
    xy = interior_points(mesh, tables)
    vals = np.asarray(u0(xy.reshape(-1, 2)), np.float64).reshape(mesh.n_elements(), tables.n_quad, 4)
    vals = np.ascontiguousarray(vals)
    out = np.empty((kEq, tables.n_p, mesh.n_elements()))
    rc = lib.dgb_project(C.byref(mesh.view), C.byref(tables.view), gas.gamma, dptr(vals), dptr(out))
    if rc == L.ERR_INADMISSIBLE:
        raise SolverAbort(L.last_message())
    _check(rc)
    return out


def project_on_device(ctx: SolverContext, u0: Callable, slot: int = L.SLOT_STATE) -> None:
    """project_initial (solver.cpp:74-97) evaluated on the device straight into a slot (the
    point values of ``u0`` are computed on the host, the projection on the GPU)."""
    xy = interior_points(ctx.mesh, ctx.tables)
    vals = np.ascontiguousarray(np.asarray(u0(xy.reshape(-1, 2)), np.float64).reshape(-1, 4))
    _check(lib.dgb_project_slot(ctx.handle, slot, dptr(vals)))


def eval_volume_pass(ctx: SolverContext, coeffs) -> np.ndarray:
    ctx.upload(L.SLOT_INPUT, coeffs)
    _check(lib.dgb_eval_volume_pass(ctx.handle, L.SLOT_INPUT))
    return ctx.download(L.SLOT_VOLUME)


def eval_surface_pass(ctx: SolverContext, coeffs, t: float, bufs: RhsBuffers = None) -> RhsBuffers:
    ctx._refresh_bc(t)
    ctx.upload(L.SLOT_INPUT, coeffs)
    _check(lib.dgb_eval_surface_pass(ctx.handle, L.SLOT_INPUT, t))
    bufs = bufs or RhsBuffers(*ctx._shape())
    sl = np.zeros((3,) + ctx._shape())
    sr = np.zeros((3,) + ctx._shape())
    _check(lib.dgb_download_surface(ctx.handle, dptr(sl), dptr(sr)))
    # slots not owned by an edge side keep their previous contents, as in the reference
    own_left = _own_left(ctx)
    bufs.surface_left[...] = np.where(own_left[:, None, None, :], sl, bufs.surface_left)
    bufs.surface_right[...] = np.where(~own_left[:, None, None, :], sr, bufs.surface_right)
    return bufs


def _own_left(ctx: SolverContext) -> np.ndarray:
    m = ctx.mesh
    ids = np.arange(m.n_elements())
    return (m.edge_left[m.elem_edge] == ids[:, None]).T  # [3][N]


def eval_rhs_pass(ctx: SolverContext, bufs: RhsBuffers) -> np.ndarray:
    ctx.upload(L.SLOT_VOLUME, bufs.volume)
    sl = np.ascontiguousarray(bufs.surface_left)
    sr = np.ascontiguousarray(bufs.surface_right)
    _check(lib.dgb_upload_surface(ctx.handle, dptr(sl), dptr(sr)))
    _check(lib.dgb_eval_rhs_pass(ctx.handle))
    return ctx.download(L.SLOT_DERIV)


def compute_rhs(ctx: SolverContext, coeffs, t: float) -> np.ndarray:
    """solver.cpp:279-284 as one fused kernel."""
    ctx._refresh_bc(t)
    ctx.upload(L.SLOT_INPUT, coeffs)
    _check(lib.dgb_compute_rhs(ctx.handle, L.SLOT_INPUT, t, L.SLOT_DERIV))
    return ctx.download(L.SLOT_DERIV)


def limit(ctx: SolverContext, coeffs: np.ndarray) -> np.ndarray:
    """solver.cpp:286-425, in place on ``coeffs`` (also returned)."""
    if ctx.tables.p != 1:
        raise ValueError("slope limiting is only supported for p = 1")
    ctx.upload(L.SLOT_INPUT, coeffs)
    _check(lib.dgb_limit(ctx.handle, L.SLOT_INPUT))
    coeffs[...] = ctx.download(L.SLOT_INPUT)
    return coeffs


def stable_dt(ctx: SolverContext, coeffs) -> float:
    ctx.upload(L.SLOT_INPUT, coeffs)
    dt = C.c_double()
    _check(lib.dgb_stable_dt(ctx.handle, L.SLOT_INPUT, ctx.options.cfl, C.byref(dt)))
    return dt.value


def _push_state(ctx: SolverContext, state: SolverState):
    ctx.upload(L.SLOT_STATE, state.coeffs)
    _check(lib.dgb_set_time(ctx.handle, state.t, state.step_count))


def _pull_state(ctx: SolverContext, state: SolverState):
    state.coeffs = ctx.download(L.SLOT_STATE)
    t, s = C.c_double(), C.c_int64()
    _check(lib.dgb_get_time(ctx.handle, C.byref(t), C.byref(s)))
    state.t, state.step_count = t.value, s.value


def _axpy(a, s, b):
    return a + s * b


def rk_step(ctx: SolverContext, state: SolverState, dt: float, op: Callable = None,
            limiting: Optional[bool] = None) -> float:
    """solver.cpp:545-557.  With ``op`` (an RhsOperator ``op(coeffs, t) -> deriv``)
    the stage algebra runs on the host around the caller's operator — the
    reference's plugin seam; without it the whole step runs on the device."""
    lim = ctx.options.limiting if limiting is None else limiting
    scheme = ctx.options.scheme_id()
    if op is None:
        if _time_dependent(ctx):
            _set_stage_tables(ctx, state.t, dt)
        _push_state(ctx, state)
        res = C.c_double()
        try:
            _check(lib.dgb_rk_step(ctx.handle, scheme, dt, int(lim), C.byref(res)))
        finally:
            _pull_state(ctx, state)
        return res.value
    u, t = state.coeffs, state.t

    def L_(c, tt):
        return np.asarray(op(c, tt))

    def lim_(c):
        return limit(ctx, c) if lim else c
    if scheme == 2:
        k1 = L_(u, t)
        s = lim_(_axpy(u, 0.5 * dt, k1))
        k2 = L_(s, t + 0.5 * dt)
        s = _axpy(u, dt, k2)
    elif scheme == 4:
        k1 = L_(u, t)
        s = lim_(_axpy(u, 0.5 * dt, k1))
        k2 = L_(s, t + 0.5 * dt)
        s = lim_(_axpy(u, 0.5 * dt, k2))
        k3 = L_(s, t + 0.5 * dt)
        s = lim_(_axpy(u, dt, k3))
        k4 = L_(s, t + dt)
        s = u + dt / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    elif scheme == 102:
        s1 = lim_(_axpy(u, dt, L_(u, t)))
        s = 0.5 * u + 0.5 * s1 + 0.5 * dt * L_(s1, t + dt)
    elif scheme == 103:
        s1 = lim_(_axpy(u, dt, L_(u, t)))
        s2 = lim_(0.75 * u + 0.25 * s1 + 0.25 * dt * L_(s1, t + dt))
        s = (1.0 / 3.0) * u + (2.0 / 3.0) * s2 + (2.0 / 3.0) * dt * L_(s2, t + 0.5 * dt)
    else:
        raise ValueError("rk_order must be 2 or 4")
    s = lim_(np.array(s))
    residual = float(np.max(np.abs(u - s))) if u.size else 0.0
    state.coeffs = s
    state.t += dt
    state.step_count += 1
    return residual


def _stage_times(scheme: int):
    n = C.c_int()
    tc = (C.c_double * 8)()
    _check(lib.dgb_scheme_stage_times(scheme, tc, C.byref(n)))
    return [tc[k] for k in range(n.value)]


def _time_dependent(ctx: SolverContext) -> bool:
    return bool(ctx.bc.time_dependent and ctx.bc.dirichlet is not None)


def _set_stage_tables(ctx: SolverContext, t: float, dt: float):
    """The Dirichlet closure at every stage time of the step (t + c_k dt), as the reference
    evaluates it inside each surface pass (solver.cpp:198-211)."""
    tabs = [ctx._bc_tables(t + ck * dt)[0] for ck in _stage_times(ctx.options.scheme_id())]
    if any(tb is None for tb in tabs):  # no boundary Gauss points (e.g. a periodic mesh)
        return
    arr = np.ascontiguousarray(np.stack(tabs))
    _check(lib.dgb_set_dirichlet_stages(ctx.handle, len(tabs), dptr(arr)))


def _host_stepped(ctx: SolverContext, state: SolverState, max_steps: int, t_end: float = None,
                  tol: float = None, on_step: Callable = None):
    """The drivers for time-dependent Dirichlet data: the step loop of solver.cpp:559-613 on the
    host (stable_dt, the stage-time tables, one device RK step), the state resident on the device.
    Returns (steps, residual)."""
    _push_state(ctx, state)
    res, dt = C.c_double(), C.c_double()
    t, s = C.c_double(), C.c_int64()
    steps, residual = 0, 0.0
    try:
        _check(lib.dgb_get_time(ctx.handle, C.byref(t), C.byref(s)))
        while steps < max_steps and (t_end is None or t.value < t_end):
            _check(lib.dgb_stable_dt(ctx.handle, L.SLOT_STATE, ctx.options.cfl, C.byref(dt)))
            h = dt.value
            if t_end is not None and t.value + h > t_end:
                h = t_end - t.value
            _set_stage_tables(ctx, t.value, h)
            _check(lib.dgb_rk_step(ctx.handle, ctx.options.scheme_id(), h, int(ctx.options.limiting), C.byref(res)))
            steps += 1
            residual = res.value
            _check(lib.dgb_get_time(ctx.handle, C.byref(t), C.byref(s)))
            if on_step:
                on_step(steps, residual)
            if tol is not None and residual <= tol:
                break
    finally:
        _pull_state(ctx, state)
    return steps, residual


def run_fixed_steps(ctx: SolverContext, state: SolverState, n_steps: int,
                    on_step: Callable = None) -> float:
    """solver.cpp:600-613 with the state resident on the device."""
    if _time_dependent(ctx):
        return _host_stepped(ctx, state, int(n_steps), on_step=on_step)[1]
    _push_state(ctx, state)
    res = C.c_double()
    hist = np.zeros(max(int(n_steps), 1))
    try:
        _check(lib.dgb_run_fixed_steps(ctx.handle, ctx.options.scheme_id(), ctx.options.cfl,
                                       int(ctx.options.limiting), int(n_steps), C.byref(res), dptr(hist)))
    finally:
        _pull_state(ctx, state)
    if on_step:
        for s in range(int(n_steps)):
            on_step(s + 1, float(hist[s]))
    return res.value


def run_to_time(ctx: SolverContext, state: SolverState, t_end: float, max_steps: int,
                on_step: Callable = None) -> float:
    """solver.cpp:581-598"""
    if _time_dependent(ctx):
        steps, residual = _host_stepped(ctx, state, int(max_steps), t_end=t_end, on_step=on_step)
        if state.t < t_end:
            raise SolverAbort(f"t_end not reached within {int(max_steps)} steps")
        return residual
    _push_state(ctx, state)
    res = C.c_double()
    steps = C.c_int64()
    cap = int(min(max_steps, 1 << 22))
    hist = np.zeros(max(cap, 1)) if on_step else None
    try:
        _check(lib.dgb_run_to_time(ctx.handle, ctx.options.scheme_id(), ctx.options.cfl,
                                   int(ctx.options.limiting), t_end, int(max_steps), C.byref(res),
                                   C.byref(steps), dptr(hist) if hist is not None else None, cap if on_step else 0))
    finally:
        _pull_state(ctx, state)
    if on_step:
        for s in range(min(steps.value, cap)):
            on_step(s + 1, float(hist[s]))
    return res.value


def run_to_steady(ctx: SolverContext, state: SolverState, tol: float, max_steps: int,
                  on_step: Callable = None) -> SteadyResult:
    """solver.cpp:559-579"""
    if _time_dependent(ctx):
        steps, residual = _host_stepped(ctx, state, int(max_steps), tol=tol, on_step=on_step)
        return SteadyResult(steps, residual, steps > 0 and residual <= tol)
    _push_state(ctx, state)
    steps, res, conv = C.c_int64(), C.c_double(), C.c_int()
    cap = int(min(max_steps, 1 << 22))
    hist = np.zeros(max(cap, 1)) if on_step else None
    try:
        _check(lib.dgb_run_to_steady(ctx.handle, ctx.options.scheme_id(), ctx.options.cfl,
                                     int(ctx.options.limiting), tol, int(max_steps), C.byref(steps),
                                     C.byref(res), C.byref(conv), dptr(hist) if hist is not None else None,
                                     cap if on_step else 0))
    finally:
        _pull_state(ctx, state)
    if on_step:
        for s in range(min(steps.value, cap)):
            on_step(s + 1, float(hist[s]))
    return SteadyResult(int(steps.value), float(res.value), bool(conv.value))


# ----------------------------------------------------------------------------- checkpoints / reductions
_MAGIC = b"DG2DCKP1"


def save_checkpoint(state: SolverState, path: str):
    """solver.cpp:615-633 (little-endian DG2DCKP1)."""
    c = np.ascontiguousarray(state.coeffs, np.float64)
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(struct.pack("<iiqdq", c.shape[0], c.shape[1], c.shape[2], state.t, state.step_count))
            f.write(c.astype("<f8").tobytes())
    except OSError:
        raise OSError(f"cannot open checkpoint file '{path}'")


def load_checkpoint(path: str) -> SolverState:
    """solver.cpp:635-660"""
    try:
        f = open(path, "rb")
    except OSError:
        raise OSError(f"cannot open checkpoint file '{path}'")
    with f:
        if f.read(8) != _MAGIC:
            raise OSError(f"'{path}' is not a dg2d checkpoint")
        hdr = f.read(struct.calcsize("<iiqdq"))
        if len(hdr) != struct.calcsize("<iiqdq"):
            raise OSError(f"corrupt checkpoint header in '{path}'")
        m, np_, n, t, step = struct.unpack("<iiqdq", hdr)
        if m <= 0 or np_ <= 0 or n <= 0:
            raise OSError(f"corrupt checkpoint header in '{path}'")
        data = np.frombuffer(f.read(8 * m * np_ * n), dtype="<f8")
        if data.size != m * np_ * n:
            raise OSError(f"truncated checkpoint '{path}'")
    return SolverState(data.reshape(m, np_, n).astype(np.float64), t, step)


def total_mass(mesh: Mesh, coeffs) -> float:
    """solver.cpp:662-670: serial element-order sum."""
    inv_sqrt2 = 1.0 / math.sqrt(2.0)
    s = 0.0
    det, c0 = mesh.det_jac, np.asarray(coeffs)[0, 0]
    for i in range(mesh.n_elements()):
        s += det[i] * c0[i] * inv_sqrt2
    return s


def compute_l2_error(ctx: SolverContext, coeffs, exact: Callable) -> float:
    """runner.cpp:127-150: L2 norm of the density error against ``exact(xy[n,2]) -> states[n,4]``
    (per-element partials on the device, summed in element order on the host)."""
    xy = interior_points(ctx.mesh, ctx.tables).reshape(-1, 2)
    rho = np.ascontiguousarray(np.asarray(exact(xy), np.float64).reshape(-1, 4)[:, 0])
    ctx.upload(L.SLOT_INPUT, coeffs)
    out = C.c_double()
    _check(lib.dgb_l2_error(ctx.handle, L.SLOT_INPUT, dptr(rho), C.byref(out)))
    return out.value


@dataclasses.dataclass
class ConvergenceRow:
    """runner.hpp ConvergenceRow"""
    mesh_letter: str
    elements: int
    error: float
    rate: Optional[float]
    steps: int


def convergence_study(p: int, letters: str = "A,B,C,D", rk_order: int = 4, cfl: float = 0.9,
                      steady_tol: float = 1e-14, max_steps: int = 5_000_000,
                      geo: "VortexGeometry" = None, gas: GasModel = GasModel(), device: Optional[int] = None):
    """runner.cpp:261-284 for the supersonic vortex (the only problem it accepts): per mesh of the
    family A.. (levels 0..), project the exact solution, run to steady state on the device,
    L2 density error, and the rate log2(e_prev / e)."""
    geo = geo or VortexGeometry()
    rows, prev = [], None
    for letter in [x for x in letters.replace(" ", "").split(",") if x]:
        level = ord(letter.upper()) - ord("A")
        mesh = generate_mesh(L.MESH_VORTEX, level, 0, geo.r_inner, geo.r_outer)
        tb = build_tables(p)
        exact = lambda xy: vortex_exact(xy, geo, gas)  # noqa: E731
        ctx = SolverContext(mesh, tb, gas=gas, bc=vortex_boundary(geo, gas),
                            options=SolverOptions(rk_order=rk_order, cfl=cfl), device=device)
        st = SolverState(project_initial(exact, mesh, tb, gas))
        sr = run_to_steady(ctx, st, steady_tol, max_steps)
        if not sr.converged:  # runner.cpp:192-194
            raise SolverAbort(f"steady run did not converge within {max_steps} steps (residual {sr.residual})")
        err = compute_l2_error(ctx, st.coeffs, exact)
        rows.append(ConvergenceRow(letter.upper(), mesh.n_elements(), err,
                                   math.log2(prev / err) if prev is not None else None, sr.steps))
        prev = err
        ctx.close()
    return rows


# ----------------------------------------------------------------------------- output (output.cpp)
def _g12(x: float) -> str:
    """std::ostream << double with precision(12) (output.cpp:22-27): printf %.12g."""
    return "%.12g" % x


def _pressure_ref(u, gamma):
    return (gamma - 1.0) * (u[..., 3] - 0.5 * (u[..., 1] * u[..., 1] + u[..., 2] * u[..., 2]) / u[..., 0])


def export_vtk(ctx: SolverContext, coeffs, path: str):
    """output.cpp:30-65: legacy VTK, 3 corner points per cell, point data rho, rho_u, rho_v, E, p;
    the corner states are evaluated on the device."""
    mesh, tb = ctx.mesh, ctx.tables
    n = mesh.n_elements()
    phic = np.ascontiguousarray([[eval_basis(tb.p, j, rs) for j in range(tb.n_p)]
                                 for rs in ((0.0, 0.0), (1.0, 0.0), (0.0, 1.0))], np.float64)
    ctx.upload(L.SLOT_INPUT, coeffs)
    st = np.empty((n, 3, 4))
    _check(lib.dgb_corner_states(ctx.handle, L.SLOT_INPUT, dptr(phic), dptr(st)))
    pr = _pressure_ref(st, ctx.gas.gamma)
    ev = mesh.elem_v
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open output file '{path}'")
    with f:
        w = f.write
        w("# vtk DataFile Version 3.0\ndg2d solution\nASCII\nDATASET UNSTRUCTURED_GRID\n")
        w(f"POINTS {3 * n} double\n")
        w("".join(f"{_g12(mesh.vx[v])} {_g12(mesh.vy[v])} 0\n" for v in ev.reshape(-1)))
        w(f"CELLS {n} {4 * n}\n")
        w("".join(f"3 {3 * i} {3 * i + 1} {3 * i + 2}\n" for i in range(n)))
        w(f"CELL_TYPES {n}\n" + "5\n" * n)
        w(f"POINT_DATA {3 * n}\n")
        for k, name in enumerate(("rho", "rho_u", "rho_v", "E", "p")):
            vals = st[:, :, k] if k < 4 else pr
            w(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
            w("".join(_g12(x) + "\n" for x in vals.reshape(-1)))


def export_csv(ctx: SolverContext, coeffs, path: str):
    """output.cpp:67-81: one row per cell: centroid, cell means (constant mode x sqrt 2), p."""
    mesh = ctx.mesh
    c = np.asarray(coeffs)
    sqrt2 = math.sqrt(2.0)
    mean = np.stack([c[m, 0] * sqrt2 for m in range(4)], 1)
    pr = _pressure_ref(mean, ctx.gas.gamma)
    ev = mesh.elem_v
    cx = (1.0 / 3.0) * (mesh.vx[ev[:, 0]] + mesh.vx[ev[:, 1]] + mesh.vx[ev[:, 2]])
    cy = (1.0 / 3.0) * (mesh.vy[ev[:, 0]] + mesh.vy[ev[:, 1]] + mesh.vy[ev[:, 2]])
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open output file '{path}'")
    with f:
        f.write("x,y,rho,rho_u,rho_v,E,p\n")
        f.write("".join(",".join(_g12(v) for v in (cx[i], cy[i], *mean[i], pr[i])) + "\n"
                        for i in range(mesh.n_elements())))


def max_abs_diff(a, b) -> float:
    """solver.cpp:672-678"""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) if a.size else 0.0
