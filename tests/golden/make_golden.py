"""Generate the golden vectors in tests/golden/ from the REAL reference solver.

Runs in the build container only (needs oracle/_ref/libdg2dref.so, built from
/root/reference/proj by oracle/Makefile).  The fixtures are small (<= 200
elements) and committed, so the CPU oracle is pinned to reference outputs on
machines where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bind  # noqa: E402

# (name, mesh kind, nx, ny, params, bc, initial-data kind, params)
CASES = [
    ("box_outflow", 0, 3, 2, (2.0, 1.0, 4), "none", 4, (7, 0.05)),
    ("sheared_reflect", 1, 3, 3, (1.1, 0.9, 0.3, 1), "none", 4, (11, 0.05)),
    ("vortex_A", 3, 0, 0, (1.0, 1.384), "vortex", 2, (1.0, 1.384, 2.25, 1.0, 1.0)),
    ("dmr_8x3", 2, 8, 3, (1.0 / 6.0,), "dmr", 3, (1.0 / 6.0, 10.0, 60.0)),
]


def make_bc(kind):
    bc = bind.RefBC()
    L = bind.ref_lib()
    if kind == "vortex":
        L.ref_bc_set_vortex(bc.h, 1.0, 1.384, 2.25, 1.0, 1.0, 1.4)
    elif kind == "dmr":
        L.ref_bc_set_double_mach(bc.h, 1.0 / 6.0, 10.0, 60.0, 1.4)
    return bc


def main():
    out = {}
    for name, kind, nx, ny, prm, bck, ick, icp in CASES:
        m = bind.RefMesh.generate(kind, nx, ny, *prm)
        out[f"{name}/dump_edges"] = np.frombuffer(m.dump_edges().encode(), dtype=np.uint8)
        for p in range(1, 6):
            if ick == 3 and p > 1:
                continue  # the projected shock is only admissible with the p=1 front cut
            t = bind.RefTables(p)
            bc = make_bc(bck)
            lim = p == 1  # steps at p = 1 run with the limiter (the DMR case needs it)
            rs = bind.RefSolver(m, t, bc, rk_order=2, cfl=0.3, limiting=lim)
            c = bind.ref_project(m, t, ick, icp)
            key = f"{name}/p{p}"
            out[key + "/coeffs"] = c
            out[key + "/volume"] = rs.volume(c)
            sl, sr = rs.surface(c, 0.0)
            out[key + "/surface_left"] = sl
            out[key + "/surface_right"] = sr
            out[key + "/rhs"] = rs.rhs(c, 0.0)
            out[key + "/stable_dt"] = np.array([rs.stable_dt(c)])
            dt = rs.stable_dt(c)
            c2, t2, r2 = rs.rk_step(c, 0.0, dt)
            out[key + "/rk2_step"] = c2
            rs.set(rk_order=4, cfl=0.3, limiting=lim)
            c4, t4, r4 = rs.rk_step(c, 0.0, dt)
            out[key + "/rk4_step"] = c4
            rs.set(rk_order=2, cfl=0.3, limiting=lim)
            cf, tf, rf, hist = rs.run_fixed_steps(c, 0.0, 10)
            out[key + "/run10"] = cf
            out[key + "/run10_t"] = np.array([tf])
            out[key + "/run10_hist"] = hist
            if p == 1:
                out[key + "/limit"] = rs.limit(c)
    np.savez_compressed(os.path.join(HERE, "reference_outputs.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
