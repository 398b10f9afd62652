"""The reference's limiter-overhead criterion (proj/tests/acceptance.cpp:368-405) on the GPU,
with both launch forms: supersonic vortex mesh C (level LEVEL, default 2), p = 1, RK2, cfl 0.9,
200 warm-up steps, STEPS timed steps with limiting off and on.  Prints one JSON line with the
event-timed ms per step of each run and the per-launch medians (stage kernel, limiter)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1601_07944_b200 import _lib as L, dg2d  # noqa: E402

level = int(os.environ.get("LEVEL", "2"))
steps = int(os.environ.get("STEPS", "10000"))
mesh = dg2d.generate_mesh(L.MESH_VORTEX, level, 0, 1.0, 1.384)
tb = dg2d.build_tables(1)
c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, tb)
stream = torch.cuda.Stream()


def samp(h, cat):
    n = C.c_int64()
    L.lib.dgb_timer_samples(h, cat, None, 0, C.byref(n))
    out = np.zeros(max(n.value, 1))
    L.lib.dgb_timer_samples(h, cat, out.ctypes.data_as(L.c_double_p), n.value, C.byref(n))
    return out[:n.value]


def run(lim, fused):
    opts = dg2d.SolverOptions(rk_order=2, cfl=0.9, limiting=lim)
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary(), options=opts)
    dg2d._check(L.lib.dgb_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    L.lib.dgb_set_fused_limiter(ctx.handle, fused)
    ctx.upload(L.SLOT_STATE, dg2d.limit(ctx, c0.copy()) if lim else c0)
    res = C.c_double()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.9, int(lim), 200, C.byref(res), None))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.9, int(lim), steps, C.byref(res), None))
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    L.lib.dgb_enable_timers(ctx.handle, 1)
    L.lib.dgb_reset_timers(ctx.handle)
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.9, int(lim), 200, C.byref(res), None))
    st, lm = samp(ctx.handle, 5), samp(ctx.handle, 3)
    ctx.close()
    return {"us_per_step": 1e3 * ms / steps, "stage_us": 1e3 * float(np.median(st)),
            "limiter_us": 1e3 * float(np.median(lm)) if lm.size else 0.0, "residual": res.value}


out = {"lib": L.LIB_PATH, "level": level, "triangles": mesh.n_elements(), "steps": steps}
off = run(False, 0)
out["off"] = off
for fused in (0, 1):
    on = run(True, fused)
    on["overhead"] = on["us_per_step"] / off["us_per_step"] - 1.0
    out["on_fused" if fused else "on_two_kernel"] = on
print(json.dumps(out))
