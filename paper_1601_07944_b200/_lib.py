"""ctypes binding of the C ABI in include/dg2d_b200/dg2d_b200.h.

Loads the in-tree ``libdg2d_b200.so`` (built by ``make`` / ``__graft_entry__.build``).
There is no fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGB_LIB") or os.path.join(_HERE, "libdg2d_b200.so")  # DGB_LIB: tuning builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the B200 path has no CPU fallback")

lib = C.CDLL(LIB_PATH)

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)


class MeshView(C.Structure):
    _fields_ = [
        ("n_vertices", C.c_int32), ("vx", c_double_p), ("vy", c_double_p),
        ("n_elements", C.c_int32), ("elem_v", c_int32_p), ("elem_edge", c_int32_p),
        ("det_jac", c_double_p), ("tau", c_double_p), ("inradius", c_double_p),
        ("n_edges", C.c_int32), ("n_boundary_edges", C.c_int32),
        ("edge_v0", c_int32_p), ("edge_v1", c_int32_p), ("edge_left", c_int32_p),
        ("edge_right", c_int32_p), ("edge_side_left", c_int32_p), ("edge_side_right", c_int32_p),
        ("edge_nx", c_double_p), ("edge_ny", c_double_p), ("edge_half_length", c_double_p),
    ]


class TablesView(C.Structure):
    _fields_ = [
        ("p", C.c_int32), ("n_p", C.c_int32), ("n_quad", C.c_int32), ("n_edge_pts", C.c_int32),
        ("phi_interior", c_double_p), ("dphi_dr_interior", c_double_p),
        ("dphi_ds_interior", c_double_p), ("w_interior", c_double_p), ("r_interior", c_double_p),
        ("phi_edge", c_double_p), ("w_edge", c_double_p), ("xi_edge", c_double_p),
        ("phi_edge_mid", c_double_p),
    ]


class BcView(C.Structure):
    _fields_ = [
        ("inflow_state", C.c_double * 4), ("dirichlet_state", c_double_p),
        ("wall_normal", c_double_p), ("has_shock", C.c_int32),
        ("shock_x0", C.c_double), ("shock_angle_deg", C.c_double), ("shock_speed", C.c_double),
        ("shock_post", C.c_double * 4), ("shock_pre", C.c_double * 4),
    ]


class PassTimers(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("volume", "surface", "rhs", "limiter", "other", "stage")]


class PartInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("rank", "world", "lo", "hi", "n_owned", "n_halo", "n_interior", "ld")] + \
        [("neighbor_mask", C.c_uint32)]


class PeerView(C.Structure):
    _fields_ = [("buf", C.c_void_p * 4), ("flags", C.c_void_p), ("scal", C.c_void_p), ("ld", C.c_int32)]


IPC_BYTES = 5 * 64


class AbortInfo(C.Structure):
    _fields_ = [("where", C.c_char * 32), ("id", C.c_int64), ("point", C.c_int32),
                ("rho", C.c_double), ("p", C.c_double)]


# status codes
OK, ERR_INADMISSIBLE, ERR_BC, ERR_ARG, ERR_CUDA, ERR_MESH, ERR_NOT_REACHED, ERR_IO = range(8)
SLOT_STATE, SLOT_INPUT, SLOT_VOLUME, SLOT_DERIV = range(4)
RK2_MIDPOINT, RK4_CLASSIC, SSP_RK2, SSP_RK3 = 2, 4, 102, 103
FLUX_LLF, FLUX_ROE = 0, 1
MESH_BOX, MESH_SHEARED_BOX, MESH_DOUBLE_MACH, MESH_VORTEX, MESH_PERIODIC_BOX = range(5)

_vp = C.c_void_p


def _sig(name, res, *args):
    if os.environ.get("DGB_LIB") and not hasattr(lib, name):
        return None  # an older tuning build (A/B timing) may lack the newest entry points
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("dgb_last_message", C.c_char_p)
_sig("dgb_create", C.c_int, C.POINTER(MeshView), C.POINTER(TablesView), C.POINTER(BcView),
     C.c_double, C.c_int, C.POINTER(_vp))
_sig("dgb_destroy", C.c_int, _vp)
_sig("dgb_set_stream", C.c_int, _vp, _vp)
_sig("dgb_set_dirichlet", C.c_int, _vp, c_double_p)
_sig("dgb_set_flux", C.c_int, _vp, C.c_int)
_sig("dgb_upload", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_download", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_upload_async", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_download_async", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_sync", C.c_int, _vp)
_sig("dgb_stage_input_async", C.c_int, _vp, c_double_p)
_sig("dgb_commit_input", C.c_int, _vp, C.c_int)
_sig("dgb_copy_slot", C.c_int, _vp, C.c_int, C.c_int)
_sig("dgb_eval_volume_pass", C.c_int, _vp, C.c_int)
_sig("dgb_eval_surface_pass", C.c_int, _vp, C.c_int, C.c_double)
_sig("dgb_download_surface", C.c_int, _vp, c_double_p, c_double_p)
_sig("dgb_upload_surface", C.c_int, _vp, c_double_p, c_double_p)
_sig("dgb_eval_rhs_pass", C.c_int, _vp)
_sig("dgb_compute_rhs", C.c_int, _vp, C.c_int, C.c_double, C.c_int)
_sig("dgb_limit", C.c_int, _vp, C.c_int)
_sig("dgb_stable_dt", C.c_int, _vp, C.c_int, C.c_double, c_double_p)
_sig("dgb_set_time", C.c_int, _vp, C.c_double, C.c_int64)
_sig("dgb_get_time", C.c_int, _vp, c_double_p, c_int64_p)
_sig("dgb_rk_step", C.c_int, _vp, C.c_int, C.c_double, C.c_int, c_double_p)
_sig("dgb_run_fixed_steps", C.c_int, _vp, C.c_int, C.c_double, C.c_int, C.c_int64, c_double_p, c_double_p)
_sig("dgb_run_to_time", C.c_int, _vp, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int64,
     c_double_p, c_int64_p, c_double_p, C.c_int64)
_sig("dgb_run_to_steady", C.c_int, _vp, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int64,
     c_int64_p, c_double_p, C.POINTER(C.c_int), c_double_p, C.c_int64)
_sig("dgb_total_mass", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_max_abs_diff", C.c_int, _vp, C.c_int, C.c_int, c_double_p)
_sig("dgb_l2_error", C.c_int, _vp, C.c_int, c_double_p, c_double_p)
_sig("dgb_corner_states", C.c_int, _vp, C.c_int, c_double_p, c_double_p)
_sig("dgb_project_slot", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_timers", C.c_int, _vp, C.POINTER(PassTimers))
_sig("dgb_reset_timers", C.c_int, _vp)
_sig("dgb_enable_timers", C.c_int, _vp, C.c_int)
_sig("dgb_last_abort", C.c_int, _vp, C.POINTER(AbortInfo))
_sig("dgb_launch_count", C.c_int64, _vp)
_sig("dgb_stage_kernel_ms", C.c_int, _vp, c_double_p, c_int64_p)
_sig("dgb_set_fused_limiter", C.c_int, _vp, C.c_int)
_sig("dgb_set_latency_forms", C.c_int, _vp, C.c_int, C.c_int)
_sig("dgb_set_trace_buffers", C.c_int, _vp, C.c_int)
_sig("dgb_set_dirichlet_stages", C.c_int, _vp, C.c_int, c_double_p)
_sig("dgb_scheme_stage_times", C.c_int, C.c_int, c_double_p, C.POINTER(C.c_int))
_sig("dgb_timer_samples", C.c_int, _vp, C.c_int, c_double_p, C.c_int64, c_int64_p)
_sig("dgb_fp64_peak", C.c_int, C.c_int, c_double_p)
_sig("dgb_part_create", C.c_int, C.POINTER(MeshView), C.POINTER(TablesView), C.POINTER(BcView),
     C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_vp))
_sig("dgb_part_plan", C.c_int, C.POINTER(MeshView), C.c_int, C.c_int, C.POINTER(PartInfo), c_int32_p, c_int32_p)
_sig("dgb_part_get_info", C.c_int, _vp, C.POINTER(PartInfo))
_sig("dgb_part_halo_ids", C.c_int, _vp, c_int32_p, c_int32_p)
_sig("dgb_part_local_ids", C.c_int, _vp, c_int32_p)
_sig("dgb_part_peer_view", C.c_int, _vp, C.POINTER(PeerView))
_sig("dgb_part_attach_peer", C.c_int, _vp, C.c_int, C.POINTER(PeerView))
_sig("dgb_part_ipc_export", C.c_int, _vp, C.c_void_p)
_sig("dgb_part_attach_peer_ipc", C.c_int, _vp, C.c_int, C.c_void_p, C.c_int32)
_sig("dgb_part_set_sends", C.c_int, _vp, C.c_int, C.c_int64, c_int32_p, c_int32_p)
_sig("dgb_part_finalize", C.c_int, _vp)
_sig("dgb_part_set_timeout", C.c_int, _vp, C.c_double)
_sig("dgb_mesh_from_msh", C.c_int, C.c_char_p, C.c_size_t, C.POINTER(_vp))
_sig("dgb_mesh_generate", C.c_int, C.c_int, C.c_int, C.c_int, c_double_p, C.c_int, C.POINTER(_vp))
_sig("dgb_mesh_generate_text", C.c_int, C.c_int, C.c_int, C.c_int, c_double_p, C.c_int,
     C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t))
_sig("dgb_mesh_get_view", C.c_int, _vp, C.POINTER(MeshView))
_sig("dgb_mesh_dump_edges", C.c_int, _vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t))
_sig("dgb_mesh_free", None, _vp)
_sig("dgb_tables_build", C.c_int, C.c_int, C.POINTER(_vp))
_sig("dgb_tables_get_view", C.c_int, _vp, C.POINTER(TablesView))
_sig("dgb_tables_free", None, _vp)
_sig("dgb_eval_basis", C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, c_double_p, c_double_p, c_double_p)
_sig("dgb_interior_points", C.c_int, C.POINTER(MeshView), C.POINTER(TablesView), c_double_p)
_sig("dgb_boundary_points", C.c_int, C.POINTER(MeshView), C.POINTER(TablesView), c_double_p)
_sig("dgb_project", C.c_int, C.POINTER(MeshView), C.POINTER(TablesView), C.c_double, c_double_p, c_double_p)
_sig("dgb_vortex_exact", C.c_int, c_double_p, C.c_int64, C.c_double, C.c_double, C.c_double,
     C.c_double, C.c_double, C.c_double, c_double_p)
_sig("dgb_rankine_hugoniot_post", C.c_int, c_double_p, C.c_double, C.c_double, C.c_double,
     C.c_double, c_double_p)
_sig("dgb_isentropic_vortex", C.c_int, c_double_p, C.c_int64, C.c_double, C.c_double, C.c_double,
     C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, c_double_p)


def last_message() -> str:
    m = lib.dgb_last_message()
    return m.decode() if m else ""


def dptr(a):
    """ctypes double* of a C-contiguous float64 numpy array."""
    return a.ctypes.data_as(c_double_p)


def iptr(a):
    return a.ctypes.data_as(c_int32_p)
