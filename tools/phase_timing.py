"""Per-phase cycle split of the DMMA stage kernel (build with -DDGB_PHASE_TIMING)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

n = int(os.environ.get("N", "708"))
mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
iv = dg2d.IsentropicVortex()
names = ["wait", "volume", "traces", "flux", "surf_proj", "epilogue"]
out = {}
for p in [int(x) for x in os.environ.get("ORDERS", "3,4,5").split(",")]:
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103))
    ctx.upload(L.SLOT_STATE, c0)
    res = C.c_double()
    f = getattr(L.lib, f"dgb_debug_phase_p{p}")
    buf = (C.c_ulonglong * 8)()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 2, C.byref(res), None))
    f(buf)
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 3, C.byref(res), None))
    f(buf)
    tot = sum(buf[i] for i in range(6))
    out[p] = {names[i]: round(buf[i] / tot, 3) for i in range(6)}
    ctx.close()
print(json.dumps(out))
