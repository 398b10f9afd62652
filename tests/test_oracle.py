"""The CPU oracle (oracle/dg2d_oracle.c) pinned against the reference:
golden vectors generated from the real reference (tests/golden/make_golden.py),
the reference itself when oracle/_ref is built, and the reference's own
known-answer tests (test_euler.cpp)."""
import math

import numpy as np
import pytest

from oracle import bind
from paper_1601_07944_b200 import _lib as L
from paper_1601_07944_b200 import dg2d

from helpers import GOLDEN, rel_per_eq, term_rel, term_scale

pytestmark = []

G = np.load(GOLDEN)
KINDS = {"box_outflow": (L.MESH_BOX, 3, 2, (2.0, 1.0, 4), "none"),
         "sheared_reflect": (L.MESH_SHEARED_BOX, 3, 3, (1.1, 0.9, 0.3, 1), "none"),
         "vortex_A": (L.MESH_VORTEX, 0, 0, (1.0, 1.384), "vortex"),
         "dmr_8x3": (L.MESH_DOUBLE_MACH, 8, 3, (1.0 / 6.0,), "dmr")}


def bc_for(kind):
    if kind == "vortex":
        return dg2d.vortex_boundary()
    if kind == "dmr":
        return dg2d.double_mach_boundary(dg2d.DoubleMachSetup())
    return dg2d.BoundaryConditions()


def golden_cases():
    out = []
    for name in KINDS:
        for p in range(1, 6):
            if f"{name}/p{p}/coeffs" in G.files:
                out.append((name, p))
    return out


@pytest.mark.parametrize("name", list(KINDS))
def test_mesh_connectivity_matches_golden_dump(name):
    kind, nx, ny, prm, _ = KINDS[name]
    mine = dg2d.generate_mesh(kind, nx, ny, *prm).dump_edges().splitlines()
    ref = G[f"{name}/dump_edges"].tobytes().decode().splitlines()
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        ia, ib = a.split()[:6], b.split()[:6]
        assert ia == ib  # identical connectivity: v0 v1 left right L R
        fa, fb = np.array(a.split()[6:], float), np.array(b.split()[6:], float)
        assert np.max(np.abs(fa - fb)) <= 4e-16


@pytest.mark.parametrize("name,p", golden_cases())
def test_oracle_matches_golden(name, p):
    kind, nx, ny, prm, bck = KINDS[name]
    mesh = dg2d.generate_mesh(kind, nx, ny, *prm)
    tb = dg2d.build_tables(p)
    orc = bind.Oracle(mesh, tb, bc_for(bck))
    key = f"{name}/p{p}"
    c = G[key + "/coeffs"]
    vol, sl, sr = G[key + "/volume"], G[key + "/surface_left"], G[key + "/surface_right"]
    scale = term_scale(vol, sl, sr, mesh.det_jac)
    v2 = orc.volume(c)
    sl2, sr2 = orc.surface(c, 0.0)
    assert rel_per_eq(v2, vol) < 1e-12
    own = (mesh.edge_left[mesh.elem_edge] == np.arange(mesh.n_elements())[:, None]).T
    assert np.max(np.abs(np.where(own[:, None, None, :], sl2 - sl, 0))) <= 1e-12 * max(np.max(np.abs(sl)), 1)
    assert np.max(np.abs(np.where(~own[:, None, None, :], sr2 - sr, 0))) <= 1e-12 * max(np.max(np.abs(sr)), 1)
    assert term_rel(orc.rhs(c, 0.0), G[key + "/rhs"], scale) <= 1e-12
    dt_ref = float(G[key + "/stable_dt"][0])
    assert abs(orc.stable_dt(c, 0.3) - dt_ref) <= 1e-13 * dt_ref
    lim = p == 1
    c2, _, _ = orc.step(c, 0.0, dt_ref, 2, lim)
    assert rel_per_eq(c2, G[key + "/rk2_step"]) <= 1e-12
    c4, _, _ = orc.step(c, 0.0, dt_ref, 4, lim)
    assert rel_per_eq(c4, G[key + "/rk4_step"]) <= 1e-12
    cf, tf, _, hist = orc.run_fixed_steps(c, 0.0, 10, 2, 0.3, lim)
    assert rel_per_eq(cf, G[key + "/run10"]) <= 1e-9
    assert abs(tf - float(G[key + "/run10_t"][0])) <= 1e-12 * tf
    if p == 1:
        assert rel_per_eq(orc.limit(c), G[key + "/limit"]) <= 1e-12


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("name", list(KINDS))
def test_oracle_matches_live_reference(name, p):
    """Same mesh arrays and the reference's own tables on both sides."""
    kind, nx, ny, prm, bck = KINDS[name]
    rm = bind.RefMesh.generate(kind, nx, ny, *prm)
    rt = bind.RefTables(p)
    mesh = dg2d.ArrayMesh(rm.export(), rm.nb)
    tb = rt.as_external()
    rbc = bind.RefBC()
    if bck == "vortex":
        bind.ref_lib().ref_bc_set_vortex(rbc.h, 1.0, 1.384, 2.25, 1.0, 1.0, 1.4)
        c = bind.ref_project(rm, rt, 2, (1.0, 1.384, 2.25, 1.0, 1.0))
    elif bck == "dmr":
        bind.ref_lib().ref_bc_set_double_mach(rbc.h, 1.0 / 6.0, 10.0, 60.0, 1.4)
        c = bind.ref_project(rm, rt, 4, (17, 0.05))
        c[:, 0] += np.array([1.4, 0.0, 0.0, 2.5])[:, None] / math.sqrt(2.0) - c[:, 0].mean(axis=1, keepdims=True)
    else:
        c = bind.ref_project(rm, rt, 1, (100 * p + 7,))
    rs = bind.RefSolver(rm, rt, rbc)
    orc = bind.Oracle(mesh, tb, bc_for(bck))
    vol = rs.volume(c)
    sl, sr = rs.surface(c, 0.05)
    scale = term_scale(vol, sl, sr, mesh.det_jac)
    assert rel_per_eq(orc.volume(c), vol) <= 1e-14
    assert term_rel(orc.rhs(c, 0.05), rs.rhs(c, 0.05), scale) <= 1e-14
    assert term_rel(orc.rhs(c, 0.05), rs.serial_rhs(c, 0.05), scale) <= 1e-13
    dt = rs.stable_dt(c)
    assert abs(orc.stable_dt(c, 0.3) - dt) <= 1e-14 * dt


@pytest.mark.skipif(not bind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scheme", [102, 103])
def test_oracle_ssp_matches_reference_composition(scheme):
    """SSP-RK2/3 are not in the reference: the oracle's schemes equal the
    composition of the reference's compute_rhs + limit."""
    rm = bind.RefMesh.generate(L.MESH_BOX, 4, 4, 1.0, 1.0, 1)
    for p, lim in [(1, True), (2, False), (4, False)]:
        rt = bind.RefTables(p)
        mesh, tb = dg2d.ArrayMesh(rm.export(), rm.nb), rt.as_external()
        rs = bind.RefSolver(rm, rt)
        c = bind.ref_project(rm, rt, 1, (31,))
        dt = rs.stable_dt(c)
        cr, tr, rr = rs.ssp_step(c, 0.0, dt, scheme, lim)
        co, to, ro = bind.Oracle(mesh, tb).step(c, 0.0, dt, scheme, lim)
        assert rel_per_eq(co, cr) <= 1e-13
        assert to == tr


# ----------------------------------------------------------------------------- KATs (test_euler.cpp)
def _o():
    return bind.oracle_lib()


def _arr(*v):
    return np.array(v, np.float64)


def test_pressure_kats():  # test_euler.cpp:26-33
    o = _o()
    assert abs(o.or_pressure(bind._d(_arr(1.0, 0, 0, 2.5)), 1.4) - 1.0) < 1e-14
    assert abs(o.or_pressure(bind._d(_arr(1.4, 0, 0, 2.5)), 1.4) - 1.0) < 1e-14
    assert abs(o.or_pressure(bind._d(_arr(1.0, 1.0, 0, 1.0)), 1.4) - 0.2) < 1e-14


def test_flux_kat():  # test_euler.cpp:61-74
    f1, f2 = np.zeros(4), np.zeros(4)
    _o().or_euler_flux(bind._d(_arr(2.0, 1.0, -1.0, 5.0)), 1.4, bind._d(f1), bind._d(f2))
    assert np.allclose(f1, [1.0, 2.3, -0.5, 3.4], rtol=1e-14, atol=0)
    assert np.allclose(f2, [-1.0, -0.5, 2.3, -3.4], rtol=1e-14, atol=0)


def test_sod_llf_kat():  # test_euler.cpp:142-153
    ul, ur = dg2d.make_state(1.0, 0, 0, 1.0), dg2d.make_state(0.125, 0, 0, 0.1)
    f = np.zeros(4)
    _o().or_llf(bind._d(ul), bind._d(ur), 1.0, 0.0, 1.4, bind._d(f))
    s = math.sqrt(1.4)
    assert abs(f[0] - (-0.5 * s * (0.125 - 1.0))) < 1e-14 * abs(f[0])
    assert abs(f[1] - 0.5 * 1.1) < 1e-14
    assert abs(f[2]) < 1e-15
    assert abs(f[3] - (-0.5 * s * (0.25 - 2.5))) < 1e-14 * abs(f[3])


def test_llf_consistency_antisymmetry_rotation():  # test_euler.cpp:84-140
    rng = np.random.default_rng(7)
    o = _o()

    def rand_state():
        return dg2d.make_state(rng.uniform(0.1, 10), rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(0.01, 10))
    for trial in range(100):
        u = rand_state()
        n = (math.cos(0.1 * trial), math.sin(0.1 * trial))
        f, f1, f2 = np.zeros(4), np.zeros(4), np.zeros(4)
        o.or_llf(bind._d(u), bind._d(u), n[0], n[1], 1.4, bind._d(f))
        o.or_euler_flux(bind._d(u), 1.4, bind._d(f1), bind._d(f2))
        scale = np.abs(n[0] * f1) + np.abs(n[1] * f2) + 1.0
        assert np.all(np.abs(f - (n[0] * f1 + n[1] * f2)) <= 1e-14 * scale)
    for _ in range(2000):
        ul, ur = rand_state(), rand_state()
        a = rng.uniform(0, 2 * math.pi)
        f, g = np.zeros(4), np.zeros(4)
        o.or_llf(bind._d(ul), bind._d(ur), math.cos(a), math.sin(a), 1.4, bind._d(f))
        o.or_llf(bind._d(ur), bind._d(ul), -math.cos(a), -math.sin(a), 1.4, bind._d(g))
        assert np.all(np.abs(f + g) <= 1e-12 * (np.abs(f) + np.abs(g) + 1))
    for trial in range(200):
        ul, ur = rand_state(), rand_state()
        th = 0.031 * trial
        c, s = math.cos(th), math.sin(th)
        rot = lambda u: np.array([u[0], c * u[1] - s * u[2], s * u[1] + c * u[2], u[3]])
        n = (0.6, 0.8)
        rn = (c * n[0] - s * n[1], s * n[0] + c * n[1])
        f, g = np.zeros(4), np.zeros(4)
        o.or_llf(bind._d(ul), bind._d(ur), n[0], n[1], 1.4, bind._d(f))
        o.or_llf(bind._d(rot(ul)), bind._d(rot(ur)), rn[0], rn[1], 1.4, bind._d(g))
        scale = abs(f[1]) + abs(f[2]) + 1
        assert abs(g[0] - f[0]) <= 1e-12 * scale
        assert abs(g[1] - (c * f[1] - s * f[2])) <= 1e-12 * scale
        assert abs(g[2] - (s * f[1] + c * f[2])) <= 1e-12 * scale


def test_post_shock_kat():  # test_euler.cpp:220-246
    dm = dg2d.DoubleMachSetup()
    post = dm.post
    assert abs(post[0] - 8.0) < 1e-13 * 8
    assert abs(float(dg2d.pressure(post)) - 116.5) < 1e-13 * 116.5
    assert abs(math.hypot(post[1] / post[0], post[2] / post[0]) - 8.25) < 1e-13 * 8.25
    assert abs(post[3] - 563.5) < 1e-13 * 563.5


# ----------------------------------------------------------------------------- Roe (not in the reference)
def _roe(ul, ur, n):
    f = np.zeros(4)
    _o().or_roe(bind._d(np.ascontiguousarray(ul, np.float64)), bind._d(np.ascontiguousarray(ur, np.float64)),
                n[0], n[1], 1.4, bind._d(f))
    return f


def _phys(u, n):
    f1, f2 = np.zeros(4), np.zeros(4)
    _o().or_euler_flux(bind._d(np.ascontiguousarray(u, np.float64)), 1.4, bind._d(f1), bind._d(f2))
    return n[0] * f1 + n[1] * f2


def test_roe_defining_properties():
    """Parity of the Roe flux is unpinned by the reference (it has only LLF); its defining
    properties pin the restatement: consistency, conservation (antisymmetry), rotational
    invariance, exact upwinding of supersonic data, and Roe's linearisation
    F(uR) - F(uL) = A~ (uR - uL) (checked through the upwind identity
    F_roe(uL,uR) = F(uL) + sum over left-running waves, i.e. the flux difference split)."""
    rng = np.random.default_rng(11)

    def rand_state():
        return dg2d.make_state(rng.uniform(0.1, 10), rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(0.01, 10))
    for trial in range(100):  # consistency F(u,u) = F(u).n
        u = rand_state()
        n = (math.cos(0.1 * trial), math.sin(0.1 * trial))
        f, ph = _roe(u, u, n), _phys(u, n)
        assert np.all(np.abs(f - ph) <= 1e-13 * (np.abs(ph) + 1))
    for _ in range(2000):  # conservation
        ul, ur = rand_state(), rand_state()
        a = rng.uniform(0, 2 * math.pi)
        f, g = _roe(ul, ur, (math.cos(a), math.sin(a))), _roe(ur, ul, (-math.cos(a), -math.sin(a)))
        assert np.all(np.abs(f + g) <= 1e-11 * (np.abs(f) + np.abs(g) + 1))
    for trial in range(200):  # rotation
        ul, ur = rand_state(), rand_state()
        th = 0.031 * trial
        c, s = math.cos(th), math.sin(th)
        rot = lambda u: np.array([u[0], c * u[1] - s * u[2], s * u[1] + c * u[2], u[3]])  # noqa: E731
        n = (0.6, 0.8)
        f, g = _roe(ul, ur, n), _roe(rot(ul), rot(ur), (c * n[0] - s * n[1], s * n[0] + c * n[1]))
        sc = abs(f[1]) + abs(f[2]) + abs(f[0]) + 1
        assert abs(g[0] - f[0]) <= 1e-11 * sc and abs(g[3] - f[3]) <= 1e-11 * (abs(f[3]) + 1)
        assert abs(g[1] - (c * f[1] - s * f[2])) <= 1e-11 * sc
        assert abs(g[2] - (s * f[1] + c * f[2])) <= 1e-11 * sc
    for _ in range(200):  # supersonic to the right: pure upwinding F = F(uL)
        rho, p = rng.uniform(0.5, 2), rng.uniform(0.5, 2)
        c = math.sqrt(1.4 * p / rho)
        ul = dg2d.make_state(rho, 3.0 * c, rng.uniform(-0.2, 0.2) * c, p)
        ur = dg2d.make_state(rho * rng.uniform(0.95, 1.05), 3.0 * c * rng.uniform(0.97, 1.03), 0.0,
                             p * rng.uniform(0.95, 1.05))
        f, ph = _roe(ul, ur, (1.0, 0.0)), _phys(ul, (1.0, 0.0))
        assert np.all(np.abs(f - ph) <= 1e-11 * (np.abs(ph) + 1))
    # contact discontinuity at rest (equal p, u = 0): the Roe flux is exactly the pressure
    ul, ur = dg2d.make_state(1.0, 0, 0, 1.0), dg2d.make_state(0.25, 0, 0, 1.0)
    f = _roe(ul, ur, (1.0, 0.0))
    assert abs(f[0]) < 1e-14 and abs(f[1] - 1.0) < 1e-14 and abs(f[2]) < 1e-14 and abs(f[3]) < 1e-14


def test_oracle_rhs_with_roe_is_conservative_and_free_stream_preserving():
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 6, 5, 10.0, 10.0)
    tb = dg2d.build_tables(3)
    u0 = dg2d.make_state(1.3, 0.4, -0.2, 0.9)
    c = dg2d.project_initial(lambda xy: np.tile(u0, (xy.shape[0], 1)), mesh, tb)
    orc = bind.Oracle(mesh, tb, flux="roe")
    d = orc.rhs(c)
    assert np.max(np.abs(d)) < 1e-12  # free stream
    c2 = dg2d.project_initial(dg2d.IsentropicVortex(), mesh, tb)
    d2 = orc.rhs(c2)
    mass = [float(np.sum(mesh.det_jac * d2[m, 0]) / math.sqrt(2.0)) for m in range(4)]
    assert max(abs(x) for x in mass) < 1e-12 * float(np.max(np.abs(d2)))  # periodic: conserved
