"""C4 workload driver for profiling: DMR 2000x500, p=1, limiter, RK2; FUSED=0|1 selects the
two-kernel or the fused stage+limiter launch; prints the per-launch medians (CUDA events)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import _lib as L, dg2d  # noqa: E402

nx = int(os.environ.get("NX", "2000"))
steps = int(os.environ.get("STEPS", "20"))
mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, nx, nx // 4, 1.0 / 6.0)
tb = dg2d.build_tables(1)
setup = dg2d.DoubleMachSetup()
bc = dg2d.double_mach_boundary(setup)
ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True))
L.lib.dgb_set_fused_limiter(ctx.handle, int(os.environ.get("FUSED", "1")))
c0 = dg2d.limit(ctx, dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb))
ctx.upload(L.SLOT_STATE, c0)
res = C.c_double()
dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.3, 1, 3, C.byref(res), None))
L.lib.dgb_enable_timers(ctx.handle, 1)
L.lib.dgb_reset_timers(ctx.handle)
dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.3, 1, steps, C.byref(res), None))


def samp(cat):
    n = C.c_int64()
    L.lib.dgb_timer_samples(ctx.handle, cat, None, 0, C.byref(n))
    out = np.zeros(max(n.value, 1))
    L.lib.dgb_timer_samples(ctx.handle, cat, out.ctypes.data_as(L.c_double_p), n.value, C.byref(n))
    return out[:n.value]


st, lm = samp(5), samp(3)
print({"fused": os.environ.get("FUSED", "1"), "stage_ms_median": float(np.median(st)),
       "limiter_ms_median": float(np.median(lm)) if lm.size else 0.0, "n": int(st.size)})
