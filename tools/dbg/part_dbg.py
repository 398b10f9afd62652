"""Debug helper: the DMR RK2 limiter case of test_in_process_partitions_bit_identical_to_whole_mesh."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
from paper_1601_07944_b200 import _lib as L, dg2d, dist as D  # noqa: E402
import test_partition as TP  # noqa: E402

world = int(os.environ.get("WORLD", "3"))
scheme = int(os.environ.get("SCHEME", "2"))
steps = int(os.environ.get("STEPS", "12"))
mesh, tb, bc, c0 = TP._problem("dmr", 1)
opts = dg2d.SolverOptions(scheme=scheme, cfl=0.3, limiting=True)
ref, res_ref = TP._whole(mesh, tb, bc, c0, opts, steps)
parts = [D.PartContext(mesh, tb, r, world, bc=bc, options=opts, device=0) for r in range(world)]
for q in parts:
    q.set_timeout(5.0)
D.connect_local(parts)
import ctypes as C  # noqa: E402
import threading  # noqa: E402
for p in parts:
    p.upload_global(L.SLOT_STATE, c0)
    dg2d._check(L.lib.dgb_set_time(p.handle, 0.0, 0))
msgs = [None] * world


def go(i):
    r = C.c_double()
    rc = L.lib.dgb_run_fixed_steps(parts[i].handle, parts[i].options.scheme_id(), 0.3, 1, 1, C.byref(r), None)
    msgs[i] = (rc, L.lib.dgb_last_message())


th = [threading.Thread(target=go, args=(i,)) for i in range(world)]
[t.start() for t in th]
[t.join() for t in th]
print("per-rank", msgs)
for s in range(1, steps + 1):
    st = dg2d.SolverState(c0.copy())
    t0 = time.time()
    try:
        res = D.run_fixed_steps_group(parts, st, s)
    except Exception as e:  # noqa: BLE001
        print("steps", s, "FAILED", e, time.time() - t0)
        break
    r1, rr = TP._whole(mesh, tb, bc, c0, opts, s)
    print("steps", s, "ok", np.array_equal(st.coeffs, r1.coeffs), np.max(np.abs(st.coeffs - r1.coeffs)), res, rr)
