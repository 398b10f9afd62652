#!/bin/bash
# compute-sanitizer passes over small cases of every kernel family (SURVEY.md section 5,
# race detection / memory safety): memcheck, racecheck (shared memory), initcheck,
# synccheck.  Output: gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1601_07944_b200 import _lib as L, dg2d, dist as D
for p in (1, 2, 3, 4, 5):
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 6, 5, 10.0, 10.0)
    tb = dg2d.build_tables(p)
    c0 = dg2d.project_initial(dg2d.IsentropicVortex(), mesh, tb)
    for flux in ("llf", "roe"):
        ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103, flux=flux))
        st = dg2d.SolverState(c0.copy())
        dg2d.run_fixed_steps(ctx, st, 2)
        dg2d.compute_rhs(ctx, c0, 0.0); dg2d.eval_volume_pass(ctx, c0); dg2d.eval_surface_pass(ctx, c0, 0.0)
        ctx.close()
    if p <= 2:  # the one-thread kernel and its trace-buffer instances (latency forms off)
        ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=103))
        L.lib.dgb_set_latency_forms(ctx.handle, 0, 0)
        dg2d.run_fixed_steps(ctx, dg2d.SolverState(c0.copy()), 3)
        ctx.close()
    # RK4 accumulator instances and the asynchronous copy path
    ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(rk_order=4))
    dg2d.run_fixed_steps(ctx, dg2d.SolverState(c0.copy()), 2)
    import ctypes as C, torch
    pin = torch.empty(c0.size, dtype=torch.float64, pin_memory=True); pin.numpy()[...] = c0.ravel()
    out = torch.empty(c0.size, dtype=torch.float64, pin_memory=True)
    ptr = lambda t: t.numpy().ctypes.data_as(L.c_double_p)
    res = C.c_double()
    dg2d._check(L.lib.dgb_upload_async(ctx.handle, L.SLOT_STATE, ptr(pin)))
    dg2d._check(L.lib.dgb_stage_input_async(ctx.handle, ptr(pin)))
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 4, 0.3, 0, 1, C.byref(res), None))
    dg2d._check(L.lib.dgb_download_async(ctx.handle, L.SLOT_STATE, ptr(out)))
    dg2d._check(L.lib.dgb_commit_input(ctx.handle, L.SLOT_STATE))
    dg2d._check(L.lib.dgb_sync(ctx.handle))
    ctx.close()
    if not os.environ.get("SAN_SKIP_PART"):  # initcheck serialises kernels: the in-process
        # partitions' spin-wait kernels would wait on peers that cannot run concurrently
        parts = [D.PartContext(mesh, tb, r, 2, options=dg2d.SolverOptions(scheme=103)) for r in range(2)]
        D.connect_local(parts)
        D.run_fixed_steps_group(parts, dg2d.SolverState(c0.copy()), 2)
dm = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, 12, 3, 1.0 / 6.0)
tb = dg2d.build_tables(1)
setup = dg2d.DoubleMachSetup()
bc = dg2d.double_mach_boundary(setup)
for fused, lat in ((-1, -1), (0, -1), (1, 0), (0, 0)):  # latency-form fused, two kernels + means, fused, one-thread
    ctx = dg2d.SolverContext(dm, tb, bc=bc, options=dg2d.SolverOptions(rk_order=2, limiting=True))
    L.lib.dgb_set_fused_limiter(ctx.handle, fused)
    L.lib.dgb_set_latency_forms(ctx.handle, lat, lat)
    c = dg2d.limit(ctx, dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), dm, tb))
    dg2d.run_fixed_steps(ctx, dg2d.SolverState(c), 2)
    ctx.close()
# time-dependent Dirichlet tables per stage (vortex mesh, inflow boundary)
vb = dg2d.vortex_boundary()
tdb = dg2d.BoundaryConditions(inflow_state=vb.inflow_state, dirichlet=lambda xy, t: vb.dirichlet(xy, t),
                              wall_normal=vb.wall_normal, time_dependent=True)
vm = dg2d.generate_mesh(L.MESH_VORTEX, 1, 0, 1.0, 1.384)
for p in (2, 3):
    tbp = dg2d.build_tables(p)
    ctx = dg2d.SolverContext(vm, tbp, bc=tdb, options=dg2d.SolverOptions(rk_order=4))
    dg2d.run_fixed_steps(ctx, dg2d.SolverState(dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), vm, tbp)), 2)
    ctx.close()
print("sanitizer case done")
PY
for tool in ${TOOLS:-memcheck racecheck initcheck synccheck}; do
  skip=""; [ $tool = initcheck ] && skip=1
  SAN_SKIP_PART=$skip timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -n 3 gpurun_out/sanitize_*.log
