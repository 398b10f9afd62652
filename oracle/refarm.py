"""TEST / BENCHMARK INFRASTRUCTURE ONLY — the reference solver's CPU arm.

Drives the UNMODIFIED reference (``oracle/_ref/libdg2dref.so``: /root/reference/proj's own
sources + the C shim ``oracle/ref_shim.cpp``, Release flags of the reference's
CMakeLists.txt:12-21 incl. ``-march=native``) through its public API only.  This module
imports nothing from the B200 package, so a process that runs the reference arm never loads
``libdg2d_b200.so``: the mesh (the periodic box, built by the reference's own
``build_connectivity`` with the hull edges joined, ``ref_mesh_periodic_box``), the tables
(``build_tables``), the initial data (``project_initial`` of Shu's isentropic vortex) and the
timed ``run_fixed_steps`` are all the reference's code.

Used by ``bench.py --impl reference`` and by the CPU column of the GPU arm.
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_NATIVE = os.path.join(HERE, "_ref", "libdg2dref.so")
_PORTABLE = os.path.join(HERE, "_ref", "libdg2dref_v3.so")
_CPU = os.path.join(HERE, "_ref", "native.cpu")

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)


def _cpu_signature() -> list:
    try:
        with open("/proc/cpuinfo") as f:
            lines = f.read().splitlines()
    except OSError:
        return []
    out = []
    for key in ("model", "flags"):
        for ln in lines:
            if ln.split(":")[0].strip() == key:
                out.append(ln.strip())
                break
    return out


# instruction-set flags of /proc/cpuinfo that -march=native code may use (the rest — hypervisor,
# mitigation and power-management bits — may differ between hosts of the same CPU model)
_ISA_PREFIXES = ("avx", "amx", "sse", "ssse", "fma", "bmi", "f16c", "movbe", "popcnt", "abm", "adx", "sha",
                 "vaes", "vpclmul", "gfni", "aes", "pclmul", "xsave", "cx16", "rdrand", "rdseed", "clwb",
                 "clflushopt", "serialize", "waitpkg", "movdir", "lzcnt", "prefetchw", "rdpid", "cldemote",
                 "pku", "ptwrite", "fsrm", "erms")


def _isa_flags(lines) -> set:
    for ln in lines:
        if ln.split(":")[0].strip() == "flags":
            return {f for f in ln.split(":", 1)[1].split() if f.startswith(_ISA_PREFIXES)}
    return set()


def ref_so_path() -> str:
    """The -march=native build when this CPU offers every instruction-set extension the build
    host had (recorded by oracle/Makefile in _ref/native.cpu), else the x86-64-v3 build."""
    if os.path.exists(_NATIVE) and os.path.exists(_CPU):
        with open(_CPU) as f:
            built = _isa_flags(f.read().splitlines())
        if built and built <= _isa_flags(_cpu_signature()):
            return _NATIVE
    return _PORTABLE if os.path.exists(_PORTABLE) else _NATIVE


def available() -> bool:
    return os.path.exists(_NATIVE) or os.path.exists(_PORTABLE)


def physical_cores() -> int:
    return len(os.sched_getaffinity(0))


_lib = None


def lib():
    """Load the reference library.  OpenMP reads its environment at load time: every host
    core, threads bound close (SURVEY.md 8(d) CPU column); torchrun exports
    OMP_NUM_THREADS=1, which would otherwise serialise the reference."""
    global _lib
    if _lib is None:
        os.environ["OMP_NUM_THREADS"] = str(physical_cores())
        # No OpenMP binding: the reference runs its passes on its own std::thread pool
        # (SolverOptions::workers), and with OMP_PROC_BIND set libgomp pins the initial thread
        # to the first place at load time, so every worker thread it spawns inherits a one-core
        # affinity (measured here: 1.2e7 vs 3.9e7 DOF-updates/s/stage on 8 cores, close/cores
        # binding vs unbound).
        for k in ("OMP_PROC_BIND", "OMP_PLACES"):
            os.environ.pop(k, None)
        L = C.CDLL(ref_so_path())
        V = C.c_void_p
        for name, res, args in [
            ("ref_last_error", C.c_char_p, []), ("ref_num_threads", C.c_int, []),
            ("ref_mesh_periodic_box", V, [C.c_int, C.c_int, C.c_double, C.c_double]),
            ("ref_mesh_free", None, [V]),
            ("ref_mesh_sizes", None, [V] + [C.POINTER(C.c_int)] * 4),
            ("ref_tables", V, [C.c_int]), ("ref_tables_free", None, [V]),
            ("ref_tables_sizes", None, [V, C.POINTER(C.c_int)]),
            ("ref_ctx_new", V, [V, V, V, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int]),
            ("ref_ctx_free", None, [V]),
            ("ref_bc_new", V, []), ("ref_bc_free", None, [V]),
            ("ref_project_isentropic_vortex", C.c_int, [V, V] + [C.c_double] * 8 + [dp]),
            ("ref_hold_set", C.c_int, [V, dp, C.c_double]),
            ("ref_hold_run_fixed_steps", C.c_int, [V, C.c_int64, dp]),
            ("ref_hold_get", C.c_int, [V, dp, dp, i64p]),
        ]:
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def n_modes(p: int) -> int:
    return (p + 1) * (p + 2) // 2


class PeriodicVortexRun:
    """One order of the benchmark workload held by the reference: periodic n x n box,
    isentropic vortex (xc = yc = 5, beta = 5, mean flow (1, 1) on the 10 x 10 box), RK2
    midpoint (the reference has no SSP-RK3; a stage costs one compute_rhs + the stage
    combination in both), CFL 0.3, all host threads."""

    def __init__(self, mesh, p: int, n_elements: int, cfl: float = 0.3):
        L = lib()
        self.p, self.N = p, n_elements
        self.tables = L.ref_tables(p)
        self.bc = L.ref_bc_new()
        self.mesh = mesh
        self.ctx = L.ref_ctx_new(mesh, self.tables, self.bc, 1.4, 2, cfl, 0, physical_cores())
        c0 = np.empty((4, n_modes(p), n_elements))
        _chk(L.ref_project_isentropic_vortex(mesh, self.tables, 1.4, 5.0, 5.0, 5.0, 1.0, 1.0, 10.0, 10.0,
                                             c0.ctypes.data_as(dp)))
        _chk(L.ref_hold_set(self.ctx, c0.ctypes.data_as(dp), 0.0))

    def run(self, steps: int) -> float:
        """`steps` RK2 steps through the reference's run_fixed_steps on the held state;
        returns the wall seconds of that one call."""
        r = C.c_double()
        t0 = time.perf_counter()
        _chk(lib().ref_hold_run_fixed_steps(self.ctx, steps, C.byref(r)))
        return time.perf_counter() - t0

    def dof_updates(self, steps: int) -> float:
        return 4.0 * n_modes(self.p) * self.N * 2 * steps

    def close(self):
        L = lib()
        if self.ctx:
            L.ref_ctx_free(self.ctx)
            L.ref_tables_free(self.tables)
            L.ref_bc_free(self.bc)
            self.ctx = None


def periodic_box(n: int):
    """(mesh handle, n_elements) of the reference-built periodic n x n box of side 10."""
    L = lib()
    m = L.ref_mesh_periodic_box(n, n, 10.0, 10.0)
    if not m:
        raise RuntimeError(L.ref_last_error().decode())
    nv, ne, ned, nb = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    L.ref_mesh_sizes(m, C.byref(nv), C.byref(ne), C.byref(ned), C.byref(nb))
    return m, ne.value


def throughput(n: int, orders, calls_per_order: int, steps_per_call: int, warmup_calls: int = 1,
               schedule=None) -> dict:
    """Best-of-`calls_per_order` seconds of one `steps_per_call`-step run_fixed_steps call per
    order (after `warmup_calls` untimed calls each), blended like the GPU arm: value = sum
    over orders of DOF updates / sum of the best seconds.  `schedule` (optional) is a list of
    orders giving the call order instead (round robin)."""
    mesh, N = periodic_box(n)
    runs = {p: PeriodicVortexRun(mesh, p, N) for p in orders}
    times = {p: [] for p in orders}
    try:
        for p in orders:
            for _ in range(warmup_calls):
                runs[p].run(steps_per_call)
        seq = schedule if schedule is not None else [p for _ in range(calls_per_order) for p in orders]
        for p in seq:
            times[p].append(runs[p].run(steps_per_call))
        for p in orders:  # every order sampled at least once
            if not times[p]:
                times[p].append(runs[p].run(steps_per_call))
        best = {p: min(times[p]) for p in orders}
        upd = {p: runs[p].dof_updates(steps_per_call) for p in orders}
    finally:
        for r in runs.values():
            r.close()
        lib().ref_mesh_free(mesh)
    return {"value": sum(upd.values()) / sum(best.values()), "N": N, "best_s": best, "all_s": times,
            "per_order": {p: upd[p] / best[p] for p in orders}, "calls": len(seq),
            "threads": lib().ref_num_threads(), "so": os.path.basename(ref_so_path())}
