"""Debug: which path (fused / two-kernel) in run mode differs from the rk_step result with the same dt."""
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
res = {}
for k, name in ((0, "fused"), (1, "two")):
    st = dg2d.SolverState(c0.copy())
    dg2d.rk_step(ctxs[k], st, dt)
    res[name + "_step"] = st.coeffs
    st = dg2d.SolverState(c0.copy())
    dg2d.run_fixed_steps(ctxs[k], st, 1)
    res[name + "_run"] = st.coeffs
    print(name, "run t", repr(st.t), "dt", repr(dt))
keys = list(res)
for a in keys:
    for b in keys:
        if a < b:
            d = np.abs(res[a] - res[b])
            print(a, b, d.max(), np.count_nonzero(d))
i = np.argwhere(np.abs(res["fused_run"] - res["two_run"]) > 0)[:5]
for m, j, e in i:
    print(m, j, e, [repr(res[k][m, j, e]) for k in keys])
