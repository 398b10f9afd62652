"""Quick GPU sanity: device passes vs the CPU oracle on small meshes, then a timing probe."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1601_07944_b200 import dg2d
from oracle import bind


def term_rel(a, b, scale):
    return max(np.max(np.abs(a[m] - b[m])) / max(np.max(scale[m]), 1e-300) for m in range(4))


worst = 0.0
for (kind, nx, ny, prm) in [(0, 3, 2, (2.0, 1.0, 4)), (1, 3, 3, (1.1, 0.9, 0.3, 1)), (2, 8, 3, (1 / 6,)),
                            (3, 0, 0, (1.0, 1.384)), (4, 4, 4, (1.0, 1.0))]:
    for p in range(1, 6):
        mesh = dg2d.generate_mesh(kind, nx, ny, *prm)
        tb = dg2d.build_tables(p)
        if kind == 3:
            bc = dg2d.vortex_boundary()
            u0 = lambda xy: dg2d.vortex_exact(xy)
        elif kind == 2:
            dm = dg2d.DoubleMachSetup()
            bc = dg2d.double_mach_boundary(dm)
            u0 = lambda xy: np.stack([1.4 + 0.2 * np.sin(xy[:, 0] + 2 * xy[:, 1]), 0.3 + 0.1 * np.cos(xy[:, 1]),
                                      -0.2 + 0.1 * np.sin(xy[:, 0]), 2.5 + 0.3 * np.cos(xy[:, 0] * xy[:, 1])], 1)
        else:
            bc = dg2d.BoundaryConditions()
            u0 = lambda xy: np.stack([1 + 0.2 * np.sin(xy[:, 0] + 2 * xy[:, 1]), 0.3 + 0.1 * np.cos(xy[:, 1]),
                                      -0.2 + 0.1 * np.sin(xy[:, 0]), 2.5 + 0.3 * np.cos(xy[:, 0] * xy[:, 1])], 1)
        c = dg2d.project_initial(u0, mesh, tb)
        ctx = dg2d.SolverContext(mesh, tb, bc=bc)
        orc = bind.Oracle(mesh, tb, bc)
        t = 0.05
        vg = dg2d.eval_volume_pass(ctx, c)
        bufs = dg2d.eval_surface_pass(ctx, c, t)
        dg = dg2d.compute_rhs(ctx, c, t)
        vo = orc.volume(c)
        slo, sro = orc.surface(c, t)
        do = orc.rhs(c, t)
        scale = (np.abs(vo) + np.abs(slo).sum(0) + np.abs(sro).sum(0)) / mesh.det_jac
        own = dg2d._own_left(ctx)
        e_v = np.max(np.abs(vg - vo)) / np.max(np.abs(vo))
        e_sl = np.max(np.abs(np.where(own[:, None, None, :], bufs.surface_left - slo, 0))) / max(np.max(np.abs(slo)), 1e-300)
        e_sr = np.max(np.abs(np.where(~own[:, None, None, :], bufs.surface_right - sro, 0))) / max(np.max(np.abs(sro)), 1e-300)
        e_r = term_rel(dg, do, scale)
        bufs.volume[...] = vg
        dg2 = dg2d.eval_rhs_pass(ctx, bufs)
        e_g = term_rel(dg2, do, scale)
        # one RK step of each scheme vs oracle
        es = [0.0]
        for scheme in ((2, 4, 102, 103) if kind != 2 else ()):
            ctx.options.scheme = scheme
            st = dg2d.SolverState(c.copy(), 0.0, 0)
            dt = dg2d.stable_dt(ctx, c)
            dto = orc.stable_dt(c, 0.3)
            res = dg2d.rk_step(ctx, st, dt)
            co, _, reso = orc.step(c, 0.0, dt, scheme)
            es.append(max(abs(dt - dto) / dto, np.max(np.abs(st.coeffs - co)) / np.max(np.abs(co)), abs(res - reso) / max(reso, 1e-300)))
        ctx.options.scheme = None
        worst = max(worst, e_v, e_r, e_g)
        print(f"kind {kind} p {p}: vol {e_v:.1e} surfL {e_sl:.1e} surfR {e_sr:.1e} rhs {e_r:.1e} gather {e_g:.1e} steps {max(es):.1e}", flush=True)
        ctx.close()
print("WORST", worst)

# limiter on a shocked field
mesh = dg2d.generate_mesh(0, 16, 4, 1.0, 0.25, 1)
tb = dg2d.build_tables(1)
sod = lambda xy: np.where((xy[:, 0] < 0.5)[:, None], dg2d.make_state(1, 0, 0, 1)[None], dg2d.make_state(0.125, 0, 0, 0.1)[None])
c = dg2d.project_initial(sod, mesh, tb)
ctx = dg2d.SolverContext(mesh, tb)
orc = bind.Oracle(mesh, tb)
lg = dg2d.limit(ctx, c.copy())
lo = orc.limit(c)
print("limiter diff", np.max(np.abs(lg - lo)))
# DMR 100 steps with limiter vs oracle
dm = dg2d.DoubleMachSetup()
mesh = dg2d.generate_mesh(2, 40, 10, 1 / 6)
bc = dg2d.double_mach_boundary(dm)
rm = bind.RefMesh.generate(2, 40, 10, 1 / 6) if bind.ref_available() else None
c = dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, dm), mesh, tb)
ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True))
orc = bind.Oracle(mesh, tb, bc)
c = orc.limit(c)
st = dg2d.SolverState(c.copy())
t0 = time.time()
dg2d.run_fixed_steps(ctx, st, 100)
co, to, ro, _ = orc.run_fixed_steps(c, 0.0, 100, 2, 0.3, True)
print("DMR 100 steps limiter: rel diff", max(np.max(np.abs(st.coeffs[m] - co[m])) / np.max(np.abs(co[m])) for m in range(4)), "t", st.t, to)

# timing probe: 1M box, each p, SSP-RK3 fixed steps
for p in range(1, 6):
    mesh = dg2d.generate_mesh(4, 708, 708, 10.0, 10.0)
    tb = dg2d.build_tables(p)
    iv = dg2d.IsentropicVortex()
    c = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103, cfl=0.3))
    st = dg2d.SolverState(c)
    dg2d.run_fixed_steps(ctx, st, 3)
    import ctypes as C
    from paper_1601_07944_b200 import _lib as L
    dg2d.lib.dgb_reset_timers(ctx.handle)
    ctx.upload(L.SLOT_STATE, c)
    t0 = time.time()
    res = C.c_double()
    L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 20, C.byref(res), None)
    wall = time.time() - t0
    ms, n = C.c_double(), C.c_int64()
    L.lib.dgb_stage_kernel_ms(ctx.handle, C.byref(ms), C.byref(n))
    dof = 4 * tb.n_p * mesh.n_elements()
    print(f"p={p}: stage kernel avg {ms.value / n.value:.3f} ms over {n.value}, DOF/s/stage {dof / (ms.value / n.value * 1e-3):.3e}, wall/step {wall / 20 * 1e3:.2f} ms")
    ctx.close()
