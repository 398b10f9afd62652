"""Per-stage wall time of run_fixed_steps vs the stage-kernel time: how much of a step is
launch gaps / per-call overhead (timers on/off, batch length)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402

mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 708, 708, 10.0, 10.0)
iv = dg2d.IsentropicVortex()
out = {}
stream = torch.cuda.Stream()
for p in [int(x) for x in os.environ.get("ORDERS", "1,3").split(",")]:
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103))
    h = ctx.handle
    dg2d._check(L.lib.dgb_set_stream(h, C.c_void_p(stream.cuda_stream)))
    ctx.upload(L.SLOT_STATE, c0)
    res = C.c_double()
    row = {}
    for timers, steps in [(1, 10), (0, 10), (0, 100), (1, 100)]:
        L.lib.dgb_enable_timers(h, timers)
        dg2d._check(L.lib.dgb_run_fixed_steps(h, 103, 0.3, 0, 3, C.byref(res), None))
        L.lib.dgb_reset_timers(h)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dg2d._check(L.lib.dgb_run_fixed_steps(h, 103, 0.3, 0, steps, C.byref(res), None))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        kms, kn = C.c_double(), C.c_int64()
        L.lib.dgb_stage_kernel_ms(h, C.byref(kms), C.byref(kn))
        row[f"timers{timers}_steps{steps}"] = {"ms_per_stage": ms / (3 * steps),
                                               "kernel_ms_per_stage": kms.value / max(kn.value, 1) if timers else None}
    out[p] = row
    ctx.close()
print(json.dumps(out, indent=1))
