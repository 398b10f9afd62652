"""Kernel time of the pass-level modes (volume only, surface only, fused RHS) per order on
the 1M periodic box: where the fused stage kernel's time goes."""
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
out = {}
for p in orders:
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb)
    ctx.upload(L.SLOT_INPUT, c0)
    h = ctx.handle
    reps = 10
    for f in (lambda: L.lib.dgb_eval_volume_pass(h, L.SLOT_INPUT), lambda: L.lib.dgb_eval_surface_pass(h, L.SLOT_INPUT, 0.0),
              lambda: L.lib.dgb_compute_rhs(h, L.SLOT_INPUT, 0.0, L.SLOT_DERIV)):
        f()
    L.lib.dgb_reset_timers(h)
    for _ in range(reps):
        dg2d._check(L.lib.dgb_eval_volume_pass(h, L.SLOT_INPUT))
        dg2d._check(L.lib.dgb_eval_surface_pass(h, L.SLOT_INPUT, 0.0))
        dg2d._check(L.lib.dgb_compute_rhs(h, L.SLOT_INPUT, 0.0, L.SLOT_DERIV))
    t = ctx.read_timers()
    out[p] = {"volume_ms": t.volume * 1e3 / reps, "surface_ms": t.surface * 1e3 / reps, "rhs_ms": t.rhs * 1e3 / reps}
    ctx.close()
print(json.dumps(out))
