"""Debug helper: in-process partitions of the periodic test mesh at p >= 3 (TMA own tiles)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
from paper_1601_07944_b200 import _lib as L, dg2d, dist as D  # noqa: E402
import test_partition as TP  # noqa: E402

p = int(os.environ.get("P", "3"))
world = int(os.environ.get("WORLD", "4"))
mesh, tb, bc, c0 = TP._problem("periodic", p)
opts = dg2d.SolverOptions(scheme=102, cfl=0.3)
ref, res_ref = TP._whole(mesh, tb, bc, c0, opts, 3)
print("whole ok", mesh.n_elements())
parts = [D.PartContext(mesh, tb, r, world, bc=bc, options=opts, device=0) for r in range(world)]
for q in parts:
    q.set_timeout(5.0)
    print("part", q.rank, q.info.n_owned, q.info.n_halo, q.info.n_interior, q.info.ld)
D.connect_local(parts)
st = dg2d.SolverState(c0.copy())
try:
    D.run_fixed_steps_group(parts, st, 3)
    print("parts", np.array_equal(st.coeffs, ref.coeffs))
except Exception as e:  # noqa: BLE001
    print("FAILED", e)
