"""Host-side setup (our mesh / basis builders) against the reference's own
tests (test_mesh.cpp, test_basis.cpp) and, when built, the reference itself."""
import math
import re

import numpy as np
import pytest

from oracle import bind
from paper_1601_07944_b200 import _lib as L
from paper_1601_07944_b200 import dg2d


@pytest.mark.parametrize("level,ne,ned", [(0, 180, 293), (1, 720, 1126), (2, 2880, 4412)])
def test_vortex_family_counts(level, ne, ned):  # test_mesh.cpp:247-255
    m = dg2d.build_connectivity(dg2d.parse_msh(dg2d.gen_vortex_msh(level)))
    assert m.n_elements() == ne and m.n_edges() == ned


@pytest.mark.parametrize("kind,nx,ny,prm", [(L.MESH_BOX, 7, 5, (2.0, 3.0, 1)),
                                            (L.MESH_SHEARED_BOX, 6, 6, (1.0, 1.0, 0.3, 1)),
                                            (L.MESH_DOUBLE_MACH, 20, 5, (1 / 6,)), (L.MESH_VORTEX, 1, 0, (1.0, 1.384))])
def test_direct_generator_equals_text_path(kind, nx, ny, prm):
    direct = dg2d.generate_mesh(kind, nx, ny, *prm)
    text = {L.MESH_BOX: lambda: dg2d.gen_box_msh(nx, ny, *prm),
            L.MESH_SHEARED_BOX: lambda: dg2d.gen_sheared_box_msh(nx, ny, *prm),
            L.MESH_DOUBLE_MACH: lambda: dg2d.gen_double_mach_msh(nx, ny, *prm),
            L.MESH_VORTEX: lambda: dg2d.gen_vortex_msh(nx)}[kind]()
    assert dg2d.build_connectivity(dg2d.parse_msh(text)).dump_edges() == direct.dump_edges()


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,nx,ny,prm", [(L.MESH_BOX, 7, 5, (2.0, 3.0, 1)),
                                            (L.MESH_SHEARED_BOX, 6, 6, (1.0, 1.0, 0.3, 1)),
                                            (L.MESH_DOUBLE_MACH, 40, 10, (1 / 6,)), (L.MESH_VORTEX, 2, 0, (1.0, 1.384))])
def test_connectivity_identical_to_reference(kind, nx, ny, prm):
    mine = dg2d.generate_mesh(kind, nx, ny, *prm)
    ref = bind.RefMesh.generate(kind, nx, ny, *prm).export()
    for k, v in ref.items():
        a = np.asarray(getattr(mine, k)).reshape(v.shape)
        if v.dtype == np.int32:
            assert np.array_equal(a, v), k
        else:
            assert np.max(np.abs(a - v)) <= 4 * np.finfo(float).eps * max(1.0, np.max(np.abs(v))), k


def test_total_area_and_determinism():  # test_mesh.cpp:225-245
    sq = dg2d.build_connectivity(dg2d.parse_msh(dg2d.two_triangle_square()))
    assert abs(sq.total_area() - 1.0) < 1e-10
    box = dg2d.build_connectivity(dg2d.parse_msh(dg2d.gen_box_msh(7, 5, 2.0, 3.0, 1)))
    assert abs(box.total_area() - 6.0) < 1e-10
    t = dg2d.gen_vortex_msh(1)
    assert dg2d.build_connectivity(dg2d.parse_msh(t)).dump_edges() == \
        dg2d.build_connectivity(dg2d.parse_msh(t)).dump_edges()


SINGLE = """$MeshFormat
2.2 0 8
$EndMeshFormat
$Nodes
3
1 0 0 0
2 1 0 0
3 0 1 0
$EndNodes
$Elements
4
1 1 2 1 1 1 2
2 1 2 1 1 2 3
3 1 2 1 1 3 1
4 2 2 10 10 1 2 3
$EndElements
"""


def test_parse_errors_carry_line_numbers():  # test_mesh.cpp:65-89
    bad = SINGLE.replace("4 2 2 10 10 1 2 3", "4 2 2 10 10 1 2 99")
    with pytest.raises(dg2d.MeshError, match=r"line 15.*undefined node 99|undefined node 99"):
        dg2d.build_connectivity(dg2d.parse_msh(bad))
    with pytest.raises(dg2d.MeshError, match="unsupported mesh format version"):
        dg2d.build_connectivity(dg2d.parse_msh(SINGLE.replace("2.2", "4.1")))
    with pytest.raises(dg2d.MeshError, match="unsupported element type"):
        dg2d.build_connectivity(dg2d.parse_msh(SINGLE.replace("4 2 2 10 10 1 2 3", "4 3 2 10 10 1 2 3")))
    m = dg2d.build_connectivity(dg2d.parse_msh(SINGLE))
    assert m.n_elements() == 1 and m.n_edges() == 3 and m.n_boundary_edges == 3


def test_untagged_hull_edge_is_rejected():  # test_mesh.cpp:264-289
    t = SINGLE.replace("4\n1 1 2 1 1 1 2\n", "3\n", 1)
    with pytest.raises(dg2d.MeshError, match="no boundary tag"):
        dg2d.build_connectivity(dg2d.parse_msh(t))


def test_periodic_box_connectivity():
    n = 6
    m = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 1.0, 1.0)
    assert m.n_elements() == 2 * n * n and m.n_edges() == 3 * n * n and m.n_boundary_edges == 0
    assert np.all(m.edge_right >= 0)
    # each element has 3 distinct neighbours and every edge is shared by exactly 2 sides
    for i in range(m.n_elements()):
        nb = {m.neighbor(i, q) for q in range(3)}
        assert len(nb) == 3 and i not in nb
    counts = np.bincount(m.elem_edge.ravel(), minlength=m.n_edges())
    assert np.all(counts == 2)
    assert abs(m.total_area() - 1.0) < 1e-12


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n", [3, 7, 40])
def test_periodic_box_identical_to_reference_built(n):
    """The reference arm's periodic box (ref_mesh_periodic_box: the reference's own
    build_connectivity with the hull edges joined) is our DGB_MESH_PERIODIC_BOX, array for
    array, and the reference's project_initial of the isentropic vortex equals ours: both
    arms of the benchmark run the identical workload."""
    mine = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
    ref = bind.RefMesh(bind.ref_lib().ref_mesh_periodic_box(n, n, 10.0, 10.0))
    assert ref.nb == 0
    for k, v in ref.export().items():
        a = np.asarray(getattr(mine, k)).reshape(v.shape)
        assert np.array_equal(a, v), k
    for p in (1, 3):
        rt = bind.RefTables(p)
        c_ref = np.empty((4, rt.n_p, ref.ne))
        assert bind.ref_lib().ref_project_isentropic_vortex(ref.h, rt.h, 1.4, 5.0, 5.0, 5.0, 1.0, 1.0, 10.0, 10.0,
                                                             c_ref.ctypes.data_as(bind.dp)) == 0
        c = dg2d.project_initial(dg2d.IsentropicVortex(), mine, dg2d.build_tables(p))
        assert np.max(np.abs(c - c_ref)) <= 1e-15 * np.max(np.abs(c_ref))


# ----------------------------------------------------------------------------- basis (test_basis.cpp)
def test_table_sizes_and_counts():
    for p, nq in zip(range(1, 6), (3, 6, 12, 16, 25)):
        t = dg2d.build_tables(p)
        assert t.n_p == (p + 1) * (p + 2) // 2 and t.n_quad == nq and t.n_edge_pts == p + 1
    t = dg2d.build_tables(5)
    stored = (t.phi_interior.size * 3 + t.phi_edge.size + t.w_interior.size + t.w_edge.size
              + t.r_interior.size + 2 * 3 * t.n_edge_pts)
    assert stored == 2070  # test_basis.cpp:158


def test_quadrature_exactness_and_orthonormality():
    fact = math.factorial
    for p in range(1, 6):
        t = dg2d.build_tables(p)
        r, s, w = t.r_interior[:, 0], t.r_interior[:, 1], t.w_interior
        assert abs(w.sum() - 0.5) < 1e-13
        for a in range(2 * p + 1):
            for b in range(2 * p + 1 - a):
                exact = fact(a) * fact(b) / fact(a + b + 2)
                assert abs(np.sum(w * r ** a * s ** b) - exact) < 1e-13
        mass = (t.phi_interior * w[:, None]).T @ t.phi_interior
        assert np.max(np.abs(mass - np.eye(t.n_p))) < 1e-10
        x, wg = t.xi_edge, t.w_edge
        for k in range(2 * p + 2):
            exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
            assert abs(np.sum(wg * x ** k) - exact) < 1e-13


def test_gradient_matches_finite_differences():  # test_basis.cpp:100-115
    h = 1e-6
    for p in (1, 3, 5):
        for j in range(dg2d.basis_count(p)):
            for rs in ((0.2, 0.3), (0.6, 0.1), (0.1, 0.7)):
                dr, ds = dg2d.eval_basis_grad(p, j, rs)
                fr = (dg2d.eval_basis(p, j, (rs[0] + h, rs[1])) - dg2d.eval_basis(p, j, (rs[0] - h, rs[1]))) / (2 * h)
                fs = (dg2d.eval_basis(p, j, (rs[0], rs[1] + h)) - dg2d.eval_basis(p, j, (rs[0], rs[1] - h))) / (2 * h)
                assert abs(dr - fr) < 1e-6 * (1 + abs(dr)) and abs(ds - fs) < 1e-6 * (1 + abs(ds))


def test_constant_mode_is_sqrt2():
    for p in range(1, 6):
        assert abs(dg2d.eval_basis(p, 0, (0.1, 0.3)) - math.sqrt(2)) < 1e-14
        assert abs(dg2d.eval_basis(p, 0, (0.0, 1.0)) - math.sqrt(2)) < 1e-14


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built")
def test_tables_match_reference():
    for p in range(1, 6):
        t, r = dg2d.build_tables(p), bind.RefTables(p)
        assert r.total_stored_doubles == {1: 68, 2: 201, 3: 544, 4: 1028, 5: 2070}[p]
        for k in ("phi_interior", "dphi_dr_interior", "dphi_ds_interior", "w_interior", "r_interior",
                  "phi_edge", "w_edge", "xi_edge", "phi_edge_mid"):
            a, b = getattr(t, k), getattr(r, k)
            assert np.max(np.abs(a - b)) <= 1e-15 * max(1.0, np.max(np.abs(b))), (p, k)


def test_projection_of_constant_and_polynomial():  # test_solver.cpp:14-47
    sq = dg2d.build_connectivity(dg2d.parse_msh(dg2d.two_triangle_square()))
    t2 = dg2d.build_tables(2)
    s = dg2d.make_state(1.3, 0.2, -0.1, 0.7)
    c = dg2d.project_initial(lambda xy: np.tile(s, (len(xy), 1)), sq, t2)
    assert np.allclose(c[:, 0], s[:, None] / math.sqrt(2), rtol=1e-14, atol=0)
    assert np.max(np.abs(c[:, 1:])) < 1e-14
    m = dg2d.generate_mesh(L.MESH_BOX, 2, 2, 1.0, 1.0, 1)
    u0 = lambda xy: np.stack([1.0 + 0.3 * xy[:, 0] - 0.2 * xy[:, 1], 0.1 + 0 * xy[:, 0], 0.2 + 0 * xy[:, 0],
                              1.0 + 0 * xy[:, 0]], 1)
    for p in (1, 3):
        t = dg2d.build_tables(p)
        c = dg2d.project_initial(u0, m, t)
        xy = dg2d.interior_points(m, t)
        rho_h = np.einsum("kj,ji->ik", t.phi_interior, c[0])
        assert np.allclose(rho_h, u0(xy.reshape(-1, 2))[:, 0].reshape(rho_h.shape), rtol=1e-12, atol=0)
    with pytest.raises(dg2d.SolverAbort, match="project_initial"):
        dg2d.project_initial(lambda xy: np.stack([np.where(xy[:, 0] < .5, 1.0, -1.0), 0 * xy[:, 0], 0 * xy[:, 0],
                                                  2.5 + 0 * xy[:, 0]], 1), m, dg2d.build_tables(1))


# ----------------------------------------------------------------------------- the C ABI boundary
def test_cabi_exports_every_declared_symbol():
    import os
    hdr = open(os.path.join(os.path.dirname(L.LIB_PATH), "..", "include", "dg2d_b200", "dg2d_b200.h")).read()
    names = set(re.findall(r"\b(dgb_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(L.lib, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_a_device():
    """The product path fails loudly when no CUDA device is present."""
    import ctypes as C
    n = C.c_int(0)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    m = dg2d.generate_mesh(L.MESH_BOX, 2, 2, 1.0, 1.0, 4)
    ctx = dg2d.SolverContext(m, dg2d.build_tables(1))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        dg2d.compute_rhs(ctx, np.zeros((4, 3, m.n_elements())), 0.0)
    del n


def test_scheme_stage_times():
    """Stage-time coefficients of each scheme (the stage k of a step runs at t + c_k dt), as the
    reference's rk_step_ws evaluates its operator (solver.cpp:513-531) and the SSP schemes."""
    import ctypes as C
    n = C.c_int()
    c = (C.c_double * 8)()
    want = {2: [0.0, 0.5], 4: [0.0, 0.5, 0.5, 1.0], 102: [0.0, 1.0], 103: [0.0, 1.0, 0.5]}
    for scheme, tc in want.items():
        assert L.lib.dgb_scheme_stage_times(scheme, c, C.byref(n)) == 0
        assert [c[k] for k in range(n.value)] == tc
    assert L.lib.dgb_scheme_stage_times(3, c, C.byref(n)) == L.ERR_ARG
