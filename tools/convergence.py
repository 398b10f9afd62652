"""Supersonic-vortex convergence study on the device (acceptance.cpp:95-146, paper Table):
meshes A-D, p=1..4, RK4, cfl 0.9, steady tol 1e-14."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_07944_b200 import dg2d  # noqa: E402

orders = [int(x) for x in os.environ.get("ORDERS", "1,2,3,4").split(",")]
letters = os.environ.get("MESHES", "A,B,C,D")
out = {}
for p in orders:
    t0 = time.time()
    rows = dg2d.convergence_study(p, letters)
    out[p] = [dict(mesh=r.mesh_letter, elements=r.elements, l2=r.error, rate=r.rate, steps=r.steps) for r in rows]
    for r in rows:
        print(f"p={p} {r.mesh_letter} {r.elements:6d} L2={r.error:.4e} rate={r.rate if r.rate is None else round(r.rate, 3)} "
              f"steps={r.steps}", flush=True)
    print(f"p={p} wall {time.time() - t0:.1f}s", flush=True)
print(json.dumps(out))
