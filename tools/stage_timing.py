"""Stage-kernel timing per order on the 1M periodic box (tuning helper)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

n = int(os.environ.get("N", "708"))
orders = [int(x) for x in os.environ.get("ORDERS", "1,2,3,4,5").split(",")]
mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
iv = dg2d.IsentropicVortex()
out = {"lib": L.LIB_PATH}
for p in orders:
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103))
    ctx.upload(L.SLOT_STATE, c0)
    res = C.c_double()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 3, C.byref(res), None))
    L.lib.dgb_reset_timers(ctx.handle)
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 10, C.byref(res), None))
    ms, k = C.c_double(), C.c_int64()
    L.lib.dgb_stage_kernel_ms(ctx.handle, C.byref(ms), C.byref(k))
    dof = 4 * tb.n_p * mesh.n_elements()
    out[p] = {"stage_ms": ms.value / k.value, "dof_per_s": dof / (ms.value / k.value * 1e-3)}
    ctx.close()
print(json.dumps(out))
