"""GPU parity: the sm_100a kernels through the C ABI against the CPU oracle and
the real reference (oracle/_ref travels to the GPU box as a built library).

Tolerances (BASELINE.json north star):
  * per RHS:  ||d_gpu - d_ref||_inf,m / ||(|vol| + sum_q |slot_q|)/detJ||_inf,m <= 1e-12
  * per run:  ||c_gpu - c_ref||_inf,m / ||c_ref||_inf,m <= 1e-9
"""
import math
import os
import tempfile

import numpy as np
import pytest

from oracle import bind
from paper_1601_07944_b200 import _lib as L
from paper_1601_07944_b200 import dg2d

from helpers import cases, owned_left, rel_per_eq, smooth_field, term_rel, term_scale

pytestmark = pytest.mark.gpu

RHS_TOL = 1e-12
RUN_TOL = 1e-9
CASES = cases()


def build(case, p, options=None):
    name, kind, nx, ny, prm, bcf, u0 = case
    mesh = dg2d.generate_mesh(kind, nx, ny, *prm)
    tb = dg2d.build_tables(p)
    bc = bcf()
    c = dg2d.project_initial(u0, mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=options or dg2d.SolverOptions())
    return mesh, tb, bc, c, ctx, bind.Oracle(mesh, tb, bc)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("ci", range(len(CASES)), ids=[c[0] for c in CASES])
def test_passes_match_oracle(ci, p):
    mesh, tb, bc, c, ctx, orc = build(CASES[ci], p)
    t = 0.05
    vol = orc.volume(c)
    sl, sr = orc.surface(c, t)
    scale = term_scale(vol, sl, sr, mesh.det_jac)
    assert rel_per_eq(dg2d.eval_volume_pass(ctx, c), vol) <= RHS_TOL
    bufs = dg2d.eval_surface_pass(ctx, c, t)
    own = owned_left(mesh)
    for q in range(3):
        for m in range(4):
            a = np.where(own[q], bufs.surface_left[q, m] - sl[q, m], bufs.surface_right[q, m] - sr[q, m])
            assert np.max(np.abs(a)) <= RHS_TOL * max(float(np.max(scale[m] * mesh.det_jac)), 1e-300)
    deriv = orc.rhs(c, t)
    assert term_rel(dg2d.compute_rhs(ctx, c, t), deriv, scale) <= RHS_TOL
    bufs.volume[...] = dg2d.eval_volume_pass(ctx, c)
    assert term_rel(dg2d.eval_rhs_pass(ctx, bufs), deriv, scale) <= RHS_TOL
    ctx.close()


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("p", [1, 3, 5])
def test_rhs_matches_live_reference_same_inputs(p):
    """The reference's own mesh arrays and tables feed the GPU; its compute_rhs is the oracle."""
    rm = bind.RefMesh.generate(L.MESH_VORTEX, 1, 0, 1.0, 1.384)
    rt = bind.RefTables(p)
    rbc = bind.RefBC()
    bind.ref_lib().ref_bc_set_vortex(rbc.h, 1.0, 1.384, 2.25, 1.0, 1.0, 1.4)
    rs = bind.RefSolver(rm, rt, rbc)
    c = bind.ref_project(rm, rt, 2, (1.0, 1.384, 2.25, 1.0, 1.0))
    mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary())
    vol = rs.volume(c)
    sl, sr = rs.surface(c, 0.0)
    scale = term_scale(vol, sl, sr, mesh.det_jac)
    assert term_rel(dg2d.compute_rhs(ctx, c, 0.0), rs.rhs(c, 0.0), scale) <= RHS_TOL
    assert abs(dg2d.stable_dt(ctx, c) - rs.stable_dt(c)) <= 1e-14 * rs.stable_dt(c)
    ctx.close()


@pytest.mark.parametrize("scheme", [2, 4, 102, 103])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_single_step_matches_oracle(scheme, p):
    mesh, tb, bc, c, ctx, orc = build(CASES[0], p, dg2d.SolverOptions(scheme=scheme))
    dt = dg2d.stable_dt(ctx, c)
    assert abs(dt - orc.stable_dt(c, 0.3)) <= 1e-14 * dt
    st = dg2d.SolverState(c.copy(), 0.25, 7)
    res = dg2d.rk_step(ctx, st, dt)
    co, to, ro = orc.step(c, 0.25, dt, scheme)
    assert rel_per_eq(st.coeffs, co) <= RHS_TOL
    assert st.t == to and st.step_count == 8
    assert abs(res - ro) <= 1e-12 * np.max(np.abs(co))
    ctx.close()


@pytest.mark.parametrize("p,scheme,steps", [(1, 2, 100), (2, 4, 50), (3, 103, 40), (5, 102, 20)])
def test_run_fixed_steps_matches_oracle(p, scheme, steps):
    mesh, tb, bc, c, ctx, orc = build(CASES[4], p, dg2d.SolverOptions(scheme=scheme))
    st = dg2d.SolverState(c.copy())
    hist = []
    dg2d.run_fixed_steps(ctx, st, steps, lambda s, r: hist.append(r))
    co, to, ro, ho = orc.run_fixed_steps(c, 0.0, steps, scheme, 0.3)
    assert rel_per_eq(st.coeffs, co) <= RUN_TOL
    assert abs(st.t - to) <= 1e-13 * to and st.step_count == steps
    assert len(hist) == steps and np.allclose(hist, ho, rtol=1e-6, atol=1e-14)
    ctx.close()


@pytest.mark.parametrize("p", [1, 2, 4])
def test_vortex_run_matches_reference(p):
    """Curved walls, Dirichlet inflow, outflow: 60 RK4 steps vs the reference's run_fixed_steps."""
    if not bind.ref_available():
        pytest.skip("oracle/_ref not built")
    rm = bind.RefMesh.generate(L.MESH_VORTEX, 1, 0, 1.0, 1.384)
    rt = bind.RefTables(p)
    rbc = bind.RefBC()
    bind.ref_lib().ref_bc_set_vortex(rbc.h, 1.0, 1.384, 2.25, 1.0, 1.0, 1.4)
    rs = bind.RefSolver(rm, rt, rbc, rk_order=4, cfl=0.9)
    c = bind.ref_project(rm, rt, 2, (1.0, 1.384, 2.25, 1.0, 1.0))
    cr, tr, rr, hr = rs.run_fixed_steps(c, 0.0, 60)
    mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary(), options=dg2d.SolverOptions(rk_order=4, cfl=0.9))
    st = dg2d.SolverState(c.copy())
    res = dg2d.run_fixed_steps(ctx, st, 60)
    assert rel_per_eq(st.coeffs, cr) <= RUN_TOL
    assert abs(st.t - tr) <= 1e-12 * tr
    assert abs(res - rr) <= 1e-12 * np.max(np.abs(cr))
    ctx.close()


def test_double_mach_with_limiter_matches_reference():
    """C4 path at desk size: DMR 200x50, p=1, limiter, RK2, 100 steps vs the reference."""
    if not bind.ref_available():
        pytest.skip("oracle/_ref not built")
    rm = bind.RefMesh.generate(L.MESH_DOUBLE_MACH, 200, 50, 1.0 / 6.0)
    rt = bind.RefTables(1)
    rbc = bind.RefBC()
    bind.ref_lib().ref_bc_set_double_mach(rbc.h, 1.0 / 6.0, 10.0, 60.0, 1.4)
    rs = bind.RefSolver(rm, rt, rbc, rk_order=2, cfl=0.3, limiting=True)
    c = rs.limit(bind.ref_project(rm, rt, 3, (1.0 / 6.0, 10.0, 60.0)))
    cr, tr, rr, _ = rs.run_fixed_steps(c, 0.0, 100)
    mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
    bc = dg2d.double_mach_boundary(dg2d.DoubleMachSetup())
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True))
    st = dg2d.SolverState(c.copy())
    dg2d.run_fixed_steps(ctx, st, 100)
    assert rel_per_eq(st.coeffs, cr) <= RUN_TOL
    assert abs(st.t - tr) <= 1e-12 * tr
    ctx.close()


def test_run_to_time_and_steady_drivers():
    mesh, tb, bc, c, ctx, orc = build(CASES[2], 2, dg2d.SolverOptions(rk_order=4, cfl=0.9))
    st = dg2d.SolverState(c.copy())
    dg2d.run_to_time(ctx, st, 0.01, 10000)
    assert st.t == 0.01
    if bind.ref_available():
        rm = bind.RefMesh.generate(L.MESH_VORTEX, 0, 0, 1.0, 1.384)
        rt = bind.RefTables(2)
        rbc = bind.RefBC()
        bind.ref_lib().ref_bc_set_vortex(rbc.h, 1.0, 1.384, 2.25, 1.0, 1.0, 1.4)
        rs = bind.RefSolver(rm, rt, rbc, rk_order=4, cfl=0.9)
        cr, tr, steps_r, _ = rs.run_to_time(c, 0.0, 0.01, 10000)
        assert st.step_count == steps_r
        assert rel_per_eq(st.coeffs, cr) <= RUN_TOL
    with pytest.raises(dg2d.SolverAbort, match="t_end not reached within 3 steps"):
        dg2d.run_to_time(ctx, dg2d.SolverState(c.copy()), 1.0, 3)
    # steady driver terminates quickly on already-steady data (test_solver.cpp:493-502)
    m2 = dg2d.generate_mesh(L.MESH_BOX, 3, 3, 1.0, 1.0, 4)
    t1 = dg2d.build_tables(1)
    u = dg2d.make_state(1.0, 0.4, 0.1, 1.0)
    c2 = dg2d.project_initial(lambda xy: np.tile(u, (len(xy), 1)), m2, t1)
    ctx2 = dg2d.SolverContext(m2, t1)
    r = dg2d.run_to_steady(ctx2, dg2d.SolverState(c2), 1e-12, 1000)
    assert r.converged and r.steps <= 2
    ctx.close()
    ctx2.close()


def test_limiter_matches_oracle_bitwise_on_shocked_data():
    m = dg2d.generate_mesh(L.MESH_BOX, 16, 4, 1.0, 0.25, 1)
    t = dg2d.build_tables(1)
    sod = lambda xy: np.where((xy[:, 0] < 0.5)[:, None], dg2d.make_state(1, 0, 0, 1)[None],
                              dg2d.make_state(0.125, 0, 0, 0.1)[None])
    c = dg2d.project_initial(sod, m, t)
    ctx = dg2d.SolverContext(m, t)
    lg = dg2d.limit(ctx, c.copy())
    lo = bind.Oracle(m, t).limit(c)
    assert np.max(np.abs(lg - lo)) <= 1e-15 * np.max(np.abs(lo))
    assert np.array_equal(lg[:, 0], c[:, 0])  # means bit-identical (test_limiter.cpp:146-158)
    with pytest.raises(ValueError, match="only supported for p = 1"):
        dg2d.limit(dg2d.SolverContext(m, dg2d.build_tables(2)), np.zeros((4, 6, m.n_elements())))
    ctx.close()


def test_free_stream_preservation():  # test_solver.cpp:231-266, acceptance.cpp:148-209
    u = dg2d.make_state(1.2, 0.8, -0.5, 1.5)
    rest = dg2d.make_state(1.2, 0.0, 0.0, 1.5)
    for p in range(1, 6):
        m = dg2d.generate_mesh(L.MESH_BOX, 3, 2, 2.0, 1.0, 4)
        t = dg2d.build_tables(p)
        c = dg2d.project_initial(lambda xy: np.tile(u, (len(xy), 1)), m, t)
        assert np.max(np.abs(dg2d.compute_rhs(dg2d.SolverContext(m, t), c, 0.0))) < 1e-11
        mv = dg2d.generate_mesh(L.MESH_VORTEX, 0, 0, 1.0, 1.384)
        bc = dg2d.BoundaryConditions(dirichlet=lambda xy, tt: np.tile(rest, (len(xy), 1)),
                                     wall_normal=lambda xy: xy / np.hypot(xy[:, 0], xy[:, 1])[:, None])
        c = dg2d.project_initial(lambda xy: np.tile(rest, (len(xy), 1)), mv, t)
        assert np.max(np.abs(dg2d.compute_rhs(dg2d.SolverContext(mv, t, bc=bc), c, 0.0))) < 1e-11


@pytest.mark.parametrize("limiting", [False, True])
def test_conservation_closed_reflecting_box(limiting):  # acceptance.cpp:240-266
    m = dg2d.generate_mesh(L.MESH_BOX, 6, 6, 1.0, 1.0, 1)
    t = dg2d.build_tables(1)

    def bump(xy):
        r2 = (xy[:, 0] - 0.5) ** 2 + (xy[:, 1] - 0.5) ** 2
        return np.stack([dg2d.make_state(1 + 0.3 * math.exp(-30 * a), 0, 0, 1 + 0.2 * math.exp(-30 * a)) for a in r2])
    c = dg2d.project_initial(bump, m, t)
    ctx = dg2d.SolverContext(m, t, options=dg2d.SolverOptions(rk_order=4, limiting=limiting))
    if limiting:
        c = dg2d.limit(ctx, c)
    mass0 = dg2d.total_mass(m, c)
    st = dg2d.SolverState(c)
    dg2d.run_fixed_steps(ctx, st, 1000)
    assert abs(dg2d.total_mass(m, st.coeffs) - mass0) / abs(mass0) < 1e-10
    ctx.close()


def test_determinism_and_bitwise_checkpoint_restart():  # test_solver.cpp:424-461
    mesh, tb, bc, c, ctx, orc = build(CASES[2], 2, dg2d.SolverOptions(rk_order=4))
    a, b = dg2d.SolverState(c.copy()), dg2d.SolverState(c.copy())
    dg2d.run_fixed_steps(ctx, a, 10)
    dg2d.run_fixed_steps(ctx, b, 10)
    assert np.array_equal(a.coeffs, b.coeffs)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ck.bin")
        dg2d.save_checkpoint(a, path)
        ld = dg2d.load_checkpoint(path)
        assert ld.t == a.t and ld.step_count == a.step_count and np.array_equal(ld.coeffs, a.coeffs)
        dg2d.run_fixed_steps(ctx, ld, 5)
        dg2d.run_fixed_steps(ctx, a, 5)
        assert np.array_equal(ld.coeffs, a.coeffs)
    ctx.close()


def test_abort_diagnostics_match_reference_semantics():  # test_solver.cpp:413-422
    m = dg2d.build_connectivity(dg2d.parse_msh(dg2d.two_triangle_square(1)))
    t = dg2d.build_tables(1)
    c = np.zeros((4, 3, 2))
    c[0, 0, :] = -1.0
    ctx = dg2d.SolverContext(m, t)
    with pytest.raises(dg2d.SolverAbort, match=r"eval_volume: inadmissible state at id 0, point 0 \(rho=-1\.414214"):
        dg2d.eval_volume_pass(ctx, c)
    # a failing step leaves the state untouched and the step counter unchanged
    good = dg2d.project_initial(smooth_field(3, 0.3), m, t)
    st = dg2d.SolverState(good.copy(), 0.0, 0)
    with pytest.raises(dg2d.SolverAbort, match="inadmissible"):
        dg2d.rk_step(ctx, st, 50.0)
    assert np.array_equal(st.coeffs, good) and st.step_count == 0 and st.t == 0.0
    with pytest.raises(ValueError, match="rk_order must be 2 or 4"):
        ctx.options.rk_order = 3
        dg2d.rk_step(ctx, st, 1e-3)
    ctx.close()


def test_custom_rhs_operator_seam():  # test_solver.cpp:351-385
    m = dg2d.build_connectivity(dg2d.parse_msh(dg2d.two_triangle_square(4)))
    t = dg2d.build_tables(1)
    for order in (2, 4):
        ctx = dg2d.SolverContext(m, t, options=dg2d.SolverOptions(rk_order=order))
        st = dg2d.SolverState(np.arange(24, dtype=float).reshape(4, 3, 2) * 0.01, 0.3)
        init = st.coeffs.copy()
        op = lambda cc, tt: 1.0 + 0.1 * np.arange(24).reshape(4, 3, 2)
        dg2d.rk_step(ctx, st, 0.25, op, False)
        assert np.allclose(st.coeffs, init + 0.25 * (1.0 + 0.1 * np.arange(24).reshape(4, 3, 2)), rtol=1e-13)
        st = dg2d.SolverState(np.zeros((4, 3, 2)), 0.3)
        dg2d.rk_step(ctx, st, 0.5, lambda cc, tt: np.full((4, 3, 2), 2.0 * tt), False)
        assert np.allclose(st.coeffs, 0.8 ** 2 - 0.3 ** 2, rtol=1e-13)


# ----------------------------------------------------------------------------- full-size properties
@pytest.mark.parametrize("p", [1, 3])
def test_full_size_free_stream_conservation_determinism(p):
    """At the benchmark size (708^2 periodic box, 1,002,528 triangles): uniform flow
    is a fixed point, mass is conserved over SSP-RK3 steps, runs are bitwise
    reproducible, and one RHS matches the CPU oracle."""
    m = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 708, 708, 10.0, 10.0)
    t = dg2d.build_tables(p)
    u = dg2d.make_state(1.0, 0.7, -0.3, 1.2)
    c = dg2d.project_initial(lambda xy: np.tile(u, (len(xy), 1)), m, t)
    ctx = dg2d.SolverContext(m, t, options=dg2d.SolverOptions(scheme=103))
    st = dg2d.SolverState(c.copy())
    dg2d.run_fixed_steps(ctx, st, 5)
    assert np.max(np.abs(st.coeffs - c)) < 1e-12
    iv = dg2d.IsentropicVortex()
    c = dg2d.project_initial(lambda xy: iv(xy), m, t)
    mass = lambda cc: math.fsum(m.det_jac * cc[0, 0] / math.sqrt(2.0))  # compensated: 1M terms
    mass0 = mass(c)
    a, b = dg2d.SolverState(c.copy()), dg2d.SolverState(c.copy())
    dg2d.run_fixed_steps(ctx, a, 5)
    dg2d.run_fixed_steps(ctx, b, 5)
    assert np.array_equal(a.coeffs, b.coeffs)
    assert abs(mass(a.coeffs) - mass0) <= 1e-13 * abs(mass0)
    if p == 1:
        orc = bind.Oracle(m, t)
        vol = orc.volume(c)
        sl, sr = orc.surface(c)
        assert term_rel(dg2d.compute_rhs(ctx, c, 0.0), orc.rhs(c), term_scale(vol, sl, sr, m.det_jac)) <= RHS_TOL
    ctx.close()


# ----------------------------------------------------------------------------- Roe flux (not in the reference)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("ci", [0, 2, 3, 4], ids=[CASES[i][0] for i in (0, 2, 3, 4)])
def test_roe_rhs_matches_oracle(ci, p):
    """The Roe option of the edge flux (north star: "Lax-Friedrichs or Roe") against the
    oracle's Roe restatement; parity unpinned by the reference (it has LLF only)."""
    name, kind, nx, ny, prm, bcf, u0 = CASES[ci]
    mesh = dg2d.generate_mesh(kind, nx, ny, *prm)
    tb = dg2d.build_tables(p)
    bc = bcf()
    c = dg2d.project_initial(u0, mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=dg2d.SolverOptions(flux="roe"))
    orc = bind.Oracle(mesh, tb, bc, flux="roe")
    vol = orc.volume(c)
    sl, sr = orc.surface(c, 0.05)
    scale = term_scale(vol, sl, sr, mesh.det_jac)
    d_roe = dg2d.compute_rhs(ctx, c, 0.05)
    assert term_rel(d_roe, orc.rhs(c, 0.05), scale) <= RHS_TOL
    # and it is a different flux from LLF
    ctx_llf = dg2d.SolverContext(mesh, tb, bc=bc)
    assert np.max(np.abs(d_roe - dg2d.compute_rhs(ctx_llf, c, 0.05))) > 1e-8
    ctx.close()
    ctx_llf.close()


@pytest.mark.parametrize("p,scheme", [(2, 103), (4, 102)])
def test_roe_run_matches_oracle(p, scheme):
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 8, 8, 10.0, 10.0)
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(dg2d.IsentropicVortex(), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=scheme, cfl=0.3, flux="roe"))
    st = dg2d.SolverState(c0.copy())
    dg2d.run_fixed_steps(ctx, st, 25)
    cr, tr, _, _ = bind.Oracle(mesh, tb, flux="roe").run_fixed_steps(c0, 0.0, 25, scheme, 0.3)
    assert rel_per_eq(st.coeffs, cr) <= RUN_TOL
    assert abs(st.t - tr) <= 1e-12 * tr
    # conservation on the periodic box is exact up to round-off
    m0, m1 = dg2d.total_mass(mesh, c0), dg2d.total_mass(mesh, st.coeffs)
    assert abs(m1 - m0) <= 1e-12 * abs(m0)
    ctx.close()


# ----------------------------------------------------------------------------- accuracy (paper table)
def test_l2_error_matches_host_restatement():
    """compute_l2_error (runner.cpp:127-150): device partials vs a host restatement."""
    mesh, tb, bc, c, ctx, orc = build(CASES[2], 3)
    exact = lambda xy: dg2d.vortex_exact(xy)  # noqa: E731
    xy = dg2d.interior_points(mesh, tb).reshape(-1, 2)
    rho_ex = exact(xy)[:, 0].reshape(mesh.n_elements(), tb.n_quad)
    phi = np.asarray(tb.view.phi_interior[:tb.n_quad * tb.n_p]).reshape(tb.n_quad, tb.n_p)
    w = np.asarray(tb.view.w_interior[:tb.n_quad])
    c2 = c * (1.0 + 1e-3 * np.sin(np.arange(c.size)).reshape(c.shape))  # not the projection itself
    rho_h = np.einsum("kj,ji->ik", phi, c2[0])
    part = mesh.det_jac * ((rho_h - rho_ex) ** 2 @ w)
    host = math.sqrt(sum(float(x) for x in part))
    dev = dg2d.compute_l2_error(ctx, c2, exact)
    assert abs(dev - host) <= 1e-13 * host
    ctx.close()


def test_convergence_rates_match_the_paper():
    """acceptance.cpp:95-146 / PAPER.md:757-785: supersonic vortex, meshes A-D, p=1..4, RK4,
    cfl 0.9, steady tolerance 1e-14; C->D rates within 0.35 of 1.910/2.953/4.086/4.983 and
    the mesh-A p=1 error within a factor 3 of 4.934e-3.  (~16 s on a B200.)"""
    expected = {1: 1.910, 2: 2.953, 3: 4.086, 4: 4.983}
    for p in (1, 2, 3, 4):
        rows = dg2d.convergence_study(p, "A,B,C,D")
        assert abs(rows[3].rate - expected[p]) <= 0.35, (p, [(r.mesh_letter, r.error, r.rate) for r in rows])
        if p == 1:
            assert 4.934e-3 / 3 <= rows[0].error <= 4.934e-3 * 3
        for a, b in zip(rows, rows[1:]):
            assert b.error < a.error


# ----------------------------------------------------------------------------- output (output.cpp)
def _read_numbers(path):
    toks, nums = [], []
    for line in open(path):
        for tok in line.replace(",", " ").split():
            try:
                nums.append(float(tok))
                toks.append("#")
            except ValueError:
                toks.append(tok)
    return toks, np.array(nums)


@pytest.mark.parametrize("fmt", ["vtk", "csv"])
def test_export_matches_reference_output(fmt, tmp_path):
    """export_vtk / export_csv (output.cpp:30-81): corner states evaluated on the device, same
    file structure and values (to the 12 printed digits) as the reference's own writer."""
    if not bind.ref_available():
        pytest.skip("oracle/_ref not built")
    rm = bind.RefMesh.generate(L.MESH_VORTEX, 1, 0, 1.0, 1.384)
    rt = bind.RefTables(2)
    c = bind.ref_project(rm, rt, 2, (1.0, 1.384, 2.25, 1.0, 1.0))
    mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary())
    ours, ref = str(tmp_path / f"ours.{fmt}"), str(tmp_path / f"ref.{fmt}")
    (dg2d.export_csv if fmt == "csv" else dg2d.export_vtk)(ctx, c, ours)
    bind.ref_export(rm, rt, c, ref, csv=(fmt == "csv"))
    ta, na = _read_numbers(ours)
    tr, nr = _read_numbers(ref)
    assert ta == tr
    assert np.all(np.abs(na - nr) <= 1e-11 * np.maximum(np.abs(nr), 1e-300))
    ctx.close()


def test_device_projection_matches_host_projection():
    """project_initial on the device (dgb_project_slot) vs the host restatement used everywhere
    else (bit-compatible with solver.cpp:74-97): equal to rounding; inadmissible data aborts."""
    for ci, p in ((2, 4), (4, 5), (3, 1)):
        name, kind, nx, ny, prm, bcf, u0 = CASES[ci]
        mesh = dg2d.generate_mesh(kind, nx, ny, *prm)
        tb = dg2d.build_tables(p)
        ctx = dg2d.SolverContext(mesh, tb, bc=bcf())
        host = dg2d.project_initial(u0, mesh, tb)
        dg2d.project_on_device(ctx, u0, L.SLOT_INPUT)
        dev = ctx.download(L.SLOT_INPUT)
        assert rel_per_eq(dev, host) <= 1e-14
        with pytest.raises(dg2d.SolverAbort, match="project_initial: inadmissible state"):
            dg2d.project_on_device(ctx, lambda xy: -np.abs(np.asarray(u0(xy))), L.SLOT_INPUT)
        ctx.close()


def test_double_mach_full_run_to_t02_matches_reference():
    """The north star's per-run bar on the paper's own case: double Mach reflection 200x50
    (dmr_desk.cfg), p=1, limiter on every stage, RK2, cfl 0.3, run to t = 0.2 (3,114 steps
    measured in SURVEY Appendix B) — identical step count, relative difference <= 1e-9."""
    if not bind.ref_available():
        pytest.skip("oracle/_ref not built")
    rm = bind.RefMesh.generate(L.MESH_DOUBLE_MACH, 200, 50, 1.0 / 6.0)
    rt = bind.RefTables(1)
    rbc = bind.RefBC()
    bind.ref_lib().ref_bc_set_double_mach(rbc.h, 1.0 / 6.0, 10.0, 60.0, 1.4)
    rs = bind.RefSolver(rm, rt, rbc, rk_order=2, cfl=0.3, limiting=True)
    c = rs.limit(bind.ref_project(rm, rt, 3, (1.0 / 6.0, 10.0, 60.0)))
    cr, tr, sr, _ = rs.run_to_time(c, 0.0, 0.2, 100_000)
    mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.double_mach_boundary(dg2d.DoubleMachSetup()),
                             options=dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True))
    st = dg2d.SolverState(c.copy())
    dg2d.run_to_time(ctx, st, 0.2, 100_000)
    assert st.step_count == sr and abs(st.t - tr) <= 1e-14
    assert rel_per_eq(st.coeffs, cr) <= RUN_TOL, rel_per_eq(st.coeffs, cr)
    m_ref, m_gpu = rs.total_mass(cr), dg2d.total_mass(mesh, st.coeffs)
    assert abs(m_gpu - m_ref) <= 1e-12 * abs(m_ref)
    ctx.close()


def test_roe_with_limiter_and_moving_shock_matches_oracle():
    """Roe flux through every boundary code of the double Mach problem (reflecting wall,
    inflow, outflow, moving shock) with the limiter on every stage, 40 RK2 steps."""
    mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, 40, 10, 1.0 / 6.0)
    tb = dg2d.build_tables(1)
    setup = dg2d.DoubleMachSetup()
    bc = dg2d.double_mach_boundary(setup)
    opts = dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True, flux="roe")
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
    c0 = dg2d.limit(ctx, dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb))
    st = dg2d.SolverState(c0.copy())
    dg2d.run_fixed_steps(ctx, st, 40)
    cr, tr, _, _ = bind.Oracle(mesh, tb, bc, flux="roe").run_fixed_steps(c0, 0.0, 40, 2, 0.3, limiting=True)
    assert rel_per_eq(st.coeffs, cr) <= RUN_TOL
    assert abs(st.t - tr) <= 1e-12 * tr
    ctx.close()


def test_async_copies_pipeline_bitwise_equal_to_synchronous():
    """dgb_upload_async / dgb_stage_input_async / dgb_commit_input / dgb_download_async /
    dgb_sync (the bench's end-to-end path): a pipelined sequence of (upload, one step,
    download) requests from pinned buffers — the next input's copy in flight while the current
    request computes and downloads — returns exactly what the synchronous calls return."""
    import ctypes as C

    import torch

    mesh, tb, bc, c, ctx, orc = build(CASES[2], 2, dg2d.SolverOptions(rk_order=2))
    h = ctx.handle
    res = C.c_double()
    inputs = [np.ascontiguousarray(c * (1.0 + 1e-3 * k)) for k in range(3)]
    want = []
    for x in inputs:  # synchronous reference: upload, one step, download
        ctx.upload(L.SLOT_STATE, x)
        dg2d._check(L.lib.dgb_run_fixed_steps(h, 2, 0.3, 0, 1, C.byref(res), None))
        want.append(ctx.download(L.SLOT_STATE))
    ctx.close()
    ctx = build(CASES[2], 2, dg2d.SolverOptions(rk_order=2))[4]  # same start time as above
    h = ctx.handle
    pins = [torch.empty(x.size, dtype=torch.float64, pin_memory=True) for x in inputs]
    outs = [torch.empty(x.size, dtype=torch.float64, pin_memory=True) for x in inputs]
    for pin, x in zip(pins, inputs):
        pin.numpy()[...] = x.ravel()
    ptr = lambda t: t.numpy().ctypes.data_as(L.c_double_p)  # noqa: E731
    # request 0 in one call; request k+1 staged (host->device copy in flight) while request k
    # computes and committed after request k's download was enqueued
    dg2d._check(L.lib.dgb_upload_async(h, L.SLOT_STATE, ptr(pins[0])))
    assert L.lib.dgb_commit_input(h, L.SLOT_STATE) == L.ERR_ARG  # nothing staged
    for k, out in enumerate(outs):
        if k + 1 < len(pins):
            dg2d._check(L.lib.dgb_stage_input_async(h, ptr(pins[k + 1])))
        dg2d._check(L.lib.dgb_run_fixed_steps(h, 2, 0.3, 0, 1, C.byref(res), None))
        dg2d._check(L.lib.dgb_download_async(h, L.SLOT_STATE, ptr(out)))
        if k + 1 < len(pins):
            dg2d._check(L.lib.dgb_commit_input(h, L.SLOT_STATE))
    dg2d._check(L.lib.dgb_sync(h))
    # staging twice without a commit is refused (the staging buffer holds one input)
    dg2d._check(L.lib.dgb_stage_input_async(h, ptr(pins[0])))
    assert L.lib.dgb_stage_input_async(h, ptr(pins[1])) == L.ERR_ARG
    dg2d._check(L.lib.dgb_commit_input(h, L.SLOT_INPUT))
    dg2d._check(L.lib.dgb_sync(h))
    for out, w in zip(outs, want):
        assert np.array_equal(out.numpy().reshape(w.shape), w)
    ctx.close()


@pytest.mark.parametrize("scheme,flux,nx", [(2, "llf", 200), (4, "llf", 120), (103, "llf", 200), (102, "roe", 120),
                                            (2, "llf", 2000)])
def test_fused_stage_limiter_bitwise_equal_to_two_kernels(scheme, flux, nx):
    """The fused stage + limiter launch (k_stage_limit: tiles taken from a counter, the limiter
    trailing through L2 behind published tiles) is bit-identical to the stage kernel followed by
    the limiter kernel, for every scheme, both fluxes, and at the C4 size (2000 x 500)."""
    mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, nx, nx // 4, 1.0 / 6.0)
    tb = dg2d.build_tables(1)
    setup = dg2d.DoubleMachSetup()
    bc = dg2d.double_mach_boundary(setup)
    opts = dg2d.SolverOptions(scheme=scheme, cfl=0.3, limiting=True, flux=flux)
    out = []
    for fused in (1, 0):
        ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
        assert L.lib.dgb_set_fused_limiter(ctx.handle, fused) == 0
        c0 = dg2d.limit(ctx, dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb))
        st = dg2d.SolverState(c0)
        res = dg2d.run_fixed_steps(ctx, st, 30 if nx < 1000 else 10)
        out.append((st.coeffs, st.t, res))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1] and out[0][2] == out[1][2]


@pytest.mark.parametrize("p,scheme,flux,limiting,mesh_kind", [
    (1, 2, "llf", True, "dmr"), (1, 4, "roe", True, "dmr"), (1, 102, "llf", True, "dmr"),
    (1, 103, "llf", False, "vortex"), (2, 103, "llf", False, "vortex"), (2, 4, "roe", False, "vortex"),
    (1, 2, "llf", False, "box")])
def test_latency_forms_bitwise_equal_to_one_thread_forms(p, scheme, flux, limiting, mesh_kind):
    """The four-lanes-per-element latency forms (stage kernel at p <= 2, limiter) chosen for small
    launches give the same bits as the one-thread forms: every scheme family, both fluxes, the
    boundary-code instance (double Mach, supersonic vortex) and a periodic box."""
    if mesh_kind == "dmr":
        mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, 120, 30, 1.0 / 6.0)
        setup = dg2d.DoubleMachSetup()
        bc = dg2d.double_mach_boundary(setup)
        u0 = lambda xy: dg2d.double_mach_initial(xy, setup)  # noqa: E731
        cfl = 0.3
    elif mesh_kind == "vortex":
        mesh = dg2d.generate_mesh(L.MESH_VORTEX, 2, 0, 1.0, 1.384)
        bc = dg2d.vortex_boundary()
        u0 = dg2d.vortex_exact
        cfl = 0.3
    else:
        mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 40, 40, 10.0, 10.0)
        bc = None
        u0 = dg2d.IsentropicVortex()
        cfl = 0.3
    tb = dg2d.build_tables(p)
    opts = dg2d.SolverOptions(scheme=scheme, cfl=cfl, limiting=limiting, flux=flux)
    out = []
    for forms in ((0, 0), (1 << 30, 1 << 30)):
        ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
        assert L.lib.dgb_set_latency_forms(ctx.handle, *forms) == 0
        assert L.lib.dgb_set_fused_limiter(ctx.handle, 0) == 0
        c0 = dg2d.project_initial(u0, mesh, tb)
        if limiting:
            c0 = dg2d.limit(ctx, c0)
        st = dg2d.SolverState(c0)
        res = dg2d.run_fixed_steps(ctx, st, 25)
        out.append((st.coeffs, st.t, res))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1] and out[0][2] == out[1][2]
    assert L.lib.dgb_set_latency_forms(None, 0, 0) == L.ERR_ARG


@pytest.mark.parametrize("scheme", [4, 103])
def test_time_dependent_dirichlet_at_every_stage_time(scheme):
    """Time-dependent boundary data inside the step: the reference evaluates its Dirichlet
    closure at every stage time (solver.cpp:198-211).  With ``time_dependent=True`` the drivers
    hand the device one table per stage (dgb_set_dirichlet_stages); the run matches the host-side
    RK around compute_rhs (the closure refreshed at each stage time) and differs from stepping
    with the table of the step's start time (what the device loop alone would do)."""
    geo, gas = dg2d.VortexGeometry(), dg2d.GasModel()

    def dirichlet(xy, t):
        s = np.array(dg2d.vortex_exact(xy, geo, gas), dtype=np.float64, copy=True)
        return s * (1.0 + 0.05 * np.sin(40.0 * t))  # rho, m, E scaled alike: admissible

    base = dg2d.vortex_boundary(geo, gas)
    bc = dg2d.BoundaryConditions(inflow_state=base.inflow_state, dirichlet=dirichlet,
                                 wall_normal=base.wall_normal, time_dependent=True)
    mesh = dg2d.generate_mesh(L.MESH_VORTEX, 1, 0, geo.r_inner, geo.r_outer)
    tb = dg2d.build_tables(2)
    c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy, geo, gas), mesh, tb)
    opts = dg2d.SolverOptions(scheme=scheme, cfl=0.3)
    steps = 8

    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
    st = dg2d.SolverState(c0.copy())
    hist = []
    res = dg2d.run_fixed_steps(ctx, st, steps, lambda s, r: hist.append(r))
    assert st.step_count == steps and len(hist) == steps and hist[-1] == res

    ref = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
    sr = dg2d.SolverState(c0.copy())
    for _ in range(steps):
        dt = dg2d.stable_dt(ref, sr.coeffs)
        dg2d.rk_step(ref, sr, dt, op=lambda c, tt: dg2d.compute_rhs(ref, c, tt))
    assert rel_per_eq(st.coeffs, sr.coeffs) <= RUN_TOL
    assert abs(st.t - sr.t) <= 1e-13 * sr.t

    stale = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
    ss = dg2d.SolverState(c0.copy())
    for _ in range(steps):
        dt = dg2d.stable_dt(stale, ss.coeffs)
        stale._refresh_bc(ss.t)  # one table, at the step's start time
        dg2d._push_state(stale, ss)
        r = __import__("ctypes").c_double()
        dg2d._check(L.lib.dgb_rk_step(stale.handle, scheme, dt, 0, __import__("ctypes").byref(r)))
        dg2d._pull_state(stale, ss)
    assert rel_per_eq(ss.coeffs, sr.coeffs) > 1e-6  # the test sees the stage times
    for c_ in (ctx, ref, stale):
        c_.close()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("scheme,flux", [(103, "llf"), (4, "llf"), (2, "roe"), (102, "llf")])
@pytest.mark.parametrize("mesh_kind", ["box", "vortex"])
def test_trace_buffers_bitwise_equal_to_interpolated_traces(p, scheme, flux, mesh_kind):
    """Trace-buffer stages (each stage writes the edge traces of its output, the next reads its own
    and its neighbours' traces, dgb_set_trace_buffers) give the same bits as interpolating every
    trace from the coefficient columns: fixed steps over several device batches, run_to_time with
    its stop rule, RK4 / SSP / midpoint, both fluxes, the boundary-code instance; p = 3, 4 take the
    packed surface, p = 5 the per-side one, p = 1, 2 the one-thread kernel (when it has trace
    instances, DGB_TRACE_P)."""
    if mesh_kind == "vortex":
        mesh = dg2d.generate_mesh(L.MESH_VORTEX, 3, 0, 1.0, 1.384)
        bc, u0 = dg2d.vortex_boundary(), dg2d.vortex_exact
    else:
        mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 41, 38, 10.0, 10.0)
        bc, u0 = None, dg2d.IsentropicVortex()
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(u0, mesh, tb)
    opts = dg2d.SolverOptions(scheme=scheme, cfl=0.3, flux=flux)
    out = []
    for tr in (0, 1):
        ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
        assert L.lib.dgb_set_trace_buffers(ctx.handle, tr) == 0
        assert L.lib.dgb_set_latency_forms(ctx.handle, 0, 0) == 0  # p <= 2: the one-thread form (trace mode)
        st = dg2d.SolverState(c0.copy())
        r1 = dg2d.run_fixed_steps(ctx, st, 9)
        r2 = dg2d.run_fixed_steps(ctx, st, 4)  # a second call: its first stage interpolates again
        t_end = st.t + 0.37 * (st.t / st.step_count) * 5
        dg2d.run_to_time(ctx, st, t_end, 1000)
        out.append((st.coeffs.copy(), st.t, st.step_count, r1, r2))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1:] == out[1][1:]
    assert L.lib.dgb_set_trace_buffers(None, 1) == L.ERR_ARG
