"""Stage-kernel median on the C3 vortex mesh (level 6, walls) with trace buffers off / on:
  P=3 python tools/dbg/c3_trace_probe.py"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
from paper_1601_07944_b200 import _lib as L, dg2d
mesh = dg2d.generate_mesh(L.MESH_VORTEX, 6, 0, 1.0, 1.384)
P = int(os.environ.get("P", "3"))
tb = dg2d.build_tables(P)
c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, tb)
out = {"p": P}
for tr in (0, 1, 0, 1):
    ctx = dg2d.SolverContext(mesh, tb, bc=dg2d.vortex_boundary(), options=dg2d.SolverOptions(scheme=103, cfl=0.3))
    L.lib.dgb_set_trace_buffers(ctx.handle, tr)
    ctx.upload(L.SLOT_STATE, c0)
    res = C.c_double()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 3, C.byref(res), None))
    L.lib.dgb_enable_timers(ctx.handle, 1); L.lib.dgb_reset_timers(ctx.handle)
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 103, 0.3, 0, 10, C.byref(res), None))
    ms, k = C.c_double(), C.c_int64()
    L.lib.dgb_stage_kernel_ms(ctx.handle, C.byref(ms), C.byref(k))
    out.setdefault(tr, []).append(ms.value / k.value)
    ctx.close()
print(json.dumps(out))
