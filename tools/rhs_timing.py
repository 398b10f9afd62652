"""RHS-kernel (kModeRhs) timing per order on the 1M periodic box: the state is not advanced,
so experimental variants that break the physics (speed-of-light skips) still time."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

n = int(os.environ.get("N", "708"))
reps = int(os.environ.get("REPS", "20"))
orders = [int(x) for x in os.environ.get("ORDERS", "1,2,3,4,5").split(",")]
mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
iv = dg2d.IsentropicVortex()
out = {"lib": L.LIB_PATH}
stream = torch.cuda.Stream()
for p in orders:
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb)
    h = ctx.handle
    dg2d._check(L.lib.dgb_set_stream(h, C.c_void_p(stream.cuda_stream)))
    ctx.upload(L.SLOT_INPUT, c0)
    for _ in range(3):
        dg2d._check(L.lib.dgb_compute_rhs(h, L.SLOT_INPUT, C.c_double(0.0), L.SLOT_DERIV))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        dg2d._check(L.lib.dgb_compute_rhs(h, L.SLOT_INPUT, C.c_double(0.0), L.SLOT_DERIV))
    e1.record(stream)
    torch.cuda.synchronize()
    out[p] = round(e0.elapsed_time(e1) / reps, 4)
    ctx.close()
print(json.dumps(out))
