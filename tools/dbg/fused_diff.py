"""Debug: fused stage+limiter vs two kernels, per step, where do they differ."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1601_07944_b200 import _lib as L, dg2d

nx = int(os.environ.get("NX", "200"))
mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, nx, nx // 4, 1.0 / 6.0)
tb = dg2d.build_tables(1)
setup = dg2d.DoubleMachSetup()
bc = dg2d.double_mach_boundary(setup)
opts = dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True)
ctxs = []
for fused in (1, 0):
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
    L.lib.dgb_set_fused_limiter(ctx.handle, fused)
    ctxs.append(ctx)
c0 = dg2d.limit(ctxs[1], dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb))
dt = dg2d.stable_dt(ctxs[1], c0)
for mode in ("rk_step", "run"):
    st = [dg2d.SolverState(c0.copy()), dg2d.SolverState(c0.copy())]
    for s in range(5):
        for k in range(2):
            if mode == "rk_step":
                dg2d.rk_step(ctxs[k], st[k], dt)
            else:
                dg2d.run_fixed_steps(ctxs[k], st[k], 1)
        d = np.abs(st[0].coeffs - st[1].coeffs)
        idx = np.argwhere(d > 0)
        print(mode, s, "maxdiff", d.max(), "ndiff", len(idx), "t", st[0].t, st[1].t,
              "elems", np.unique(idx[:, 2])[:20] if len(idx) else [], "modes", np.unique(idx[:, 1]) if len(idx) else [])
