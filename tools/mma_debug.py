"""Tiny DMMA-kernel probe: one volume / surface / rhs pass at p on a small periodic box."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1601_07944_b200 import _lib as L  # noqa: E402
from paper_1601_07944_b200 import dg2d  # noqa: E402
from oracle import bind  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
tb = dg2d.build_tables(p)
c0 = dg2d.project_initial(dg2d.IsentropicVortex(), mesh, tb)
ctx = dg2d.SolverContext(mesh, tb, device=0)
orc = bind.Oracle(mesh, tb)
for name, f, g in [("volume", lambda: dg2d.eval_volume_pass(ctx, c0), lambda: orc.volume(c0)),
                   ("rhs", lambda: dg2d.compute_rhs(ctx, c0, 0.0), lambda: orc.rhs(c0, 0.0))]:
    t0 = time.time()
    a = f()
    b = g()
    print(name, "max abs diff %.3e" % np.max(np.abs(a - b)), "max |ref| %.3e" % np.max(np.abs(b)),
          "%.2fs" % (time.time() - t0), flush=True)
