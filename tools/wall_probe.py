"""Wall time per RK stage of whole device step loops (CUDA events around dgb_run_fixed_steps,
no per-kernel timers), small and large meshes, plus the reference's limiter-overhead workload:
what the launch path (gaps between the dependent kernels of a step) costs.  Prints one JSON line.
  DGB_LIB=... ORDERS=1,3 python tools/wall_probe.py"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

stream = torch.cuda.Stream()
orders = [int(x) for x in os.environ.get("ORDERS", "1,2,3,4,5").split(",")]
out = {"lib": L.LIB_PATH}


def timed(ctx, scheme, cfl, lim, steps):
    res = C.c_double()
    h = ctx.handle
    dg2d._check(L.lib.dgb_set_stream(h, C.c_void_p(stream.cuda_stream)))
    dg2d._check(L.lib.dgb_run_fixed_steps(h, scheme, cfl, lim, max(steps // 10, 3), C.byref(res), None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    dg2d._check(L.lib.dgb_run_fixed_steps(h, scheme, cfl, lim, steps, C.byref(res), None))
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


iv = dg2d.IsentropicVortex()
for n, steps in ((38, 2000), (708, 20)):
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
    for p in orders:
        tb = dg2d.build_tables(p)
        c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
        ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103))
        ctx.upload(L.SLOT_STATE, c0)
        out[f"box{n}_p{p}_us_per_stage"] = timed(ctx, 103, 0.3, 0, steps) * 1e3 / (3 * steps)
        ctx.close()
# the reference's limiter-overhead workload (acceptance.cpp:368-405): vortex mesh C, p=1, RK2
mesh = dg2d.generate_mesh(L.MESH_VORTEX, 2, 0, 1.0, 1.384)
tb = dg2d.build_tables(1)
c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, tb)
t = {}
for lim in (0, 1):
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary(),
                             options=dg2d.SolverOptions(rk_order=2, cfl=0.9, limiting=bool(lim)))
    ctx.upload(L.SLOT_STATE, dg2d.limit(ctx, c0.copy()) if lim else c0)
    t[lim] = timed(ctx, 2, 0.9, lim, 4000)
    ctx.close()
out["meshC_off_us_per_step"] = t[0] * 1e3 / 4000
out["meshC_on_us_per_step"] = t[1] * 1e3 / 4000
out["meshC_overhead"] = (t[1] - t[0]) / t[0]
print(json.dumps(out))
