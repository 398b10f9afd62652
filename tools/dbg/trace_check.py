"""Trace-buffer stage instances vs interpolated traces: max |difference| of the state after a few
steps (p = 3, 4; periodic box and the vortex mesh with walls; SSP-RK3, RK4, midpoint RK2)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

iv = dg2d.IsentropicVortex()
cases = [("box", dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 40, 37, 10.0, 10.0), None, lambda xy: iv(xy)),
         ("vortex", dg2d.generate_mesh(L.MESH_VORTEX, 3, 0, 1.0, 1.384), dg2d.vortex_boundary(),
          lambda xy: dg2d.vortex_exact(xy))]
worst = 0.0
for name, mesh, bc, f in cases:
    for p in (3, 4):
        tb = dg2d.build_tables(p)
        c0 = dg2d.project_initial(f, mesh, tb)
        for opts in (dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3), dg2d.SolverOptions(rk_order=4, cfl=0.3),
                     dg2d.SolverOptions(rk_order=2, cfl=0.3)):
            out = []
            for tr in (0, 1):
                ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts)
                dg2d._check(L.lib.dgb_set_trace_buffers(ctx.handle, tr))
                st = dg2d.SolverState(c0.copy())
                dg2d.run_fixed_steps(ctx, st, 7)
                out.append((st.coeffs.copy(), st.t, st.step_count))
                ctx.close()
            d = float(np.max(np.abs(out[0][0] - out[1][0])))
            worst = max(worst, d)
            print(name, p, opts, "maxdiff", d, "t", out[0][1], out[1][1])
print("WORST", worst)
