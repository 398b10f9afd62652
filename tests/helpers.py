"""Shared builders for the parity tests (test infrastructure)."""
import os

import numpy as np

from paper_1601_07944_b200 import _lib as L
from paper_1601_07944_b200 import dg2d

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_outputs.npz")


def smooth_field(seed, amp=0.2):
    """acceptance.cpp:41-49 style smooth admissible field (vectorised)."""
    a1, a2, ph = 0.7 + 0.13 * (seed % 7), 1.1 + 0.09 * (seed % 5), 0.31 * (seed % 11)

    def f(xy):
        s1 = np.sin(a1 * xy[:, 0] + a2 * xy[:, 1] + ph)
        s2 = np.sin(a2 * xy[:, 0] - a1 * xy[:, 1] + 2 * ph)
        rho, u, v, p = 1.0 + amp * 1.1 * s1, 1.5 * amp * s2, 1.25 * amp * s1, 1.0 + amp * s2
        return np.stack([rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)], 1)
    return f


# (name, mesh kind, nx, ny, params, boundary conditions factory, initial data factory)
def cases():
    dm = dg2d.DoubleMachSetup()
    mild_dmr = lambda xy: np.stack([1.4 + 0.1 * np.sin(xy[:, 0] + 2 * xy[:, 1]), 0.2 + 0.05 * np.cos(xy[:, 1]),
                                    -0.1 + 0.05 * np.sin(xy[:, 0]), 2.6 + 0.1 * np.cos(xy[:, 0] * xy[:, 1])], 1)
    return [
        ("box_outflow", L.MESH_BOX, 3, 2, (2.0, 1.0, 4), lambda: dg2d.BoundaryConditions(), smooth_field(3)),
        ("sheared_reflect", L.MESH_SHEARED_BOX, 3, 3, (1.1, 0.9, 0.3, 1), lambda: dg2d.BoundaryConditions(),
         smooth_field(5)),
        ("vortex_A", L.MESH_VORTEX, 0, 0, (1.0, 1.384), lambda: dg2d.vortex_boundary(), lambda xy: dg2d.vortex_exact(xy)),
        ("dmr_8x3", L.MESH_DOUBLE_MACH, 8, 3, (1.0 / 6.0,), lambda: dg2d.double_mach_boundary(dm), mild_dmr),
        ("periodic_4", L.MESH_PERIODIC_BOX, 4, 4, (10.0, 10.0), lambda: dg2d.BoundaryConditions(),
         lambda xy: dg2d.IsentropicVortex()(xy)),
    ]


def term_scale(vol, sl, sr, det):
    """(|vol| + sum_q |slot_q|) / detJ, per coefficient."""
    return (np.abs(vol) + np.abs(sl).sum(0) + np.abs(sr).sum(0)) / det


def term_rel(a, b, scale):
    """Per-equation max |a - b| / max term scale (the per-RHS parity metric)."""
    return max(float(np.max(np.abs(a[m] - b[m]))) / max(float(np.max(scale[m])), 1e-300) for m in range(4))


def rel_per_eq(a, b):
    """Per-equation max |a - b| / max |b| (the per-run parity metric)."""
    return max(float(np.max(np.abs(a[m] - b[m]))) / max(float(np.max(np.abs(b[m]))), 1e-300) for m in range(4))


def owned_left(mesh):
    ids = np.arange(mesh.n_elements())
    return (mesh.edge_left[mesh.elem_edge] == ids[:, None]).T
