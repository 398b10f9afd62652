#!/usr/bin/env python
"""Benchmark: FP64 DOF-updates/s per RK stage of the B200 modal-DG Euler path.

Workload (BASELINE.json configs[1], at the >=1M-triangle size the metric names):
periodic isentropic vortex on a 708x708 box split into 1,002,528 triangles,
orders p = 1..5 swept, SSP-RK3 (3 stages per step), CFL 0.3, random-free
synthetic initial data.  A bench "step" is one full RK time step at every
order of the sweep; `value` = sum over orders of 4*Np*N*stages*K / sum of the
device time of the timed regions (CUDA events on the solver stream).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): weak scaling.  The periodic box grows to n x (n*world)
cells, every rank owns a contiguous strip of 2 n^2 triangles and exchanges the
halo elements with its neighbours every stage through peer memory (the stage
kernel stores them into the peer's halo columns).  Device
time is the max over ranks; `value` counts the DOF updates of all ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

SCHEMES = {"ssp3": (103, 3), "ssp2": (102, 2), "rk2": (2, 2), "rk4": (4, 4)}
NQ = {1: 3, 2: 6, 3: 12, 4: 16, 5: 25}
METRIC = "FP64 DOF-updates/sec per RK stage (Euler, p=1-5)"


def np_(p):
    return (p + 1) * (p + 2) // 2


def alg_bytes(p, e):
    """bytes per element per stage (read stage, read u^n, write; geometry)."""
    return 24 * 4 * np_(p) + 40 + 34 * e


def alg_flops(p, e):
    """minimal FLOPs per element per stage (FMA = 2)."""
    n = np_(p)
    return NQ[p] * (24 * n + 52) + e * (p + 1) * (32 * n + 115) + 24 * n


def ncu_traffic(p):
    """DRAM bytes per stage-kernel launch measured by ncu (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(HERE, "profiles", "traffic.json")) as f:
            return float(json.load(f)["bytes_per_launch"][str(p)])
    except Exception:
        return None


def measured_peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling during the timed region (pynvml)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop, self._t = period, threading.Event(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n_gpus, same_device=False):
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    pg = None
    if same_device:  # test mode: every rank on cuda:0 (gloo; NCCL refuses duplicate GPUs)
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return rank, world, local, pg


def max_over_ranks(x, pg, local):
    if pg is None:
        return x
    import torch
    dev = f"cuda:{local}" if pg.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


# ----------------------------------------------------------------------------- our arm
def samples(h, category):
    """Per-launch device ms of a timer category (3 limiter, 5 stage kernel) since the reset."""
    from paper_1601_07944_b200 import _lib as L
    n = C.c_int64()
    L.lib.dgb_timer_samples(h, category, None, 0, C.byref(n))
    out = np.zeros(max(n.value, 1))
    L.lib.dgb_timer_samples(h, category, out.ctypes.data_as(L.c_double_p), n.value, C.byref(n))
    return out[:n.value]


def timed_run(h, stream, scheme, cfl, limiting, steps, pg=None, local=0, kernel_stages=100, stages=3):
    """Device-timed runs of the resident solver (dgb_run_fixed_steps):
      * throughput pass: exactly `steps` steps, no per-kernel events (an event record costs
        ~4 us of GPU time between kernels, tools/gap_probe.py), CUDA events on the launch
        stream around the whole call, max over ranks;
      * kernel pass: enough steps for >= `kernel_stages` stages with CUDA events around every
        stage-kernel (and limiter) launch on the same stream; the medians come from it.
    Returns (ms of the throughput pass, launches in it, stage-kernel ms samples, limiter ms samples)."""
    import torch
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    res = C.c_double()

    def one(n, timers):
        L.lib.dgb_enable_timers(h, timers)
        L.lib.dgb_reset_timers(h)
        l0 = L.lib.dgb_launch_count(h)
        barrier(pg)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        dg2d._check(L.lib.dgb_run_fixed_steps(h, scheme, cfl, int(limiting), n, C.byref(res), None))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(pg)
        return max_over_ranks(ev0.elapsed_time(ev1), pg, local), L.lib.dgb_launch_count(h) - l0

    ms, launches = one(steps, 0)
    one(max(steps, -(-kernel_stages // stages)), 1)
    st, lim = samples(h, 5), samples(h, 3)
    L.lib.dgb_enable_timers(h, 0)
    return ms, launches, st, lim


def roofline(p, e_ratio, n_elem, kernel_ms, hbm_gbs, fp64_tf, extra_bytes=0.0):
    """SURVEY.md 8(d) algorithmic bytes / flops per element per stage x elements, over the
    median stage-kernel duration; the binding roof is the larger of the two times."""
    b = alg_bytes(p, e_ratio) * n_elem + extra_bytes
    f = alg_flops(p, e_ratio) * n_elem
    bound = "hbm" if b / (hbm_gbs * 1e9) >= f / (fp64_tf * 1e12) else "fp64"
    ach = b / (kernel_ms * 1e-3) / 1e9 if bound == "hbm" else f / (kernel_ms * 1e-3) / 1e12
    peak = hbm_gbs if bound == "hbm" else fp64_tf
    return {"bound": bound, "achieved": ach, "peak": peak, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
            "frac": ach / peak, "traffic": ncu_traffic(p), "kernel_ms": kernel_ms,
            "alg_bytes_per_launch": b, "alg_flops_per_launch": f}


def run_b200(args, rank, world, local, pg):
    import torch
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d

    from paper_1601_07944_b200 import dist as D

    torch.cuda.set_device(local)
    scheme, stages = SCHEMES[args.scheme]
    orders = [int(x) for x in args.orders.split(",")]
    n = args.n
    # weak scaling: the periodic box grows with the rank count (n x n*world cells), every
    # rank owns a contiguous strip of 2 n^2 triangles and exchanges halo edges with its
    # two neighbours every stage
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n * world, 10.0, 10.0 * world)
    N_glob = mesh.n_elements()
    N = N_glob // world
    e_ratio = mesh.n_edges() / N_glob
    iv = dg2d.IsentropicVortex()
    hbm_gbs, hbm_src = measured_peaks()
    fp64 = C.c_double()
    dg2d._check(L.lib.dgb_fp64_peak(local, C.byref(fp64)))
    fp64_tf = fp64.value

    per_order, tot_dof_upd, tot_ms, tot_launch = [], 0.0, 0.0, 0
    e2e_dof, e2e_ms, h2d, d2h = 0.0, 0.0, 0, 0
    stream = torch.cuda.Stream(device=local)
    sampler = ClockSampler(local)
    legs = {}
    with sampler:
        for p in orders:
            tb = dg2d.build_tables(p)
            opts = dg2d.SolverOptions(scheme=scheme, cfl=args.cfl)
            if world > 1:
                ctx = D.PartContext(mesh, tb, rank, world, options=opts, device=local)
                D.connect_process_group(ctx)
                c0 = D.project_local(ctx, lambda xy: iv(xy))
            else:
                ctx = dg2d.SolverContext(mesh, tb, options=opts, device=local)
                c0 = dg2d.project_initial(lambda xy: iv(xy), mesh, tb)
            h = ctx.handle
            dg2d._check(L.lib.dgb_set_stream(h, C.c_void_p(stream.cuda_stream)))
            ctx.upload(L.SLOT_STATE, c0)
            res = C.c_double()
            dg2d._check(L.lib.dgb_run_fixed_steps(h, scheme, args.cfl, 0, args.warmup, C.byref(res), None))
            ms, launches, st_ms, _ = timed_run(h, stream, scheme, args.cfl, False, args.steps, pg, local,
                                               stages=stages)
            k_med = float(np.median(st_ms))
            dof = 4 * np_(p) * N_glob
            upd = dof * stages * args.steps
            roof = roofline(p, e_ratio, N, k_med, hbm_gbs, fp64_tf)
            per_order.append({"p": p, "value": upd / (ms * 1e-3), "ms_per_step": ms / args.steps,
                              "stage_kernel_ms_median": k_med, "stage_kernel_ms_mean": float(np.mean(st_ms)),
                              "stage_kernel_samples": int(st_ms.size),
                              "kernel_share": float(np.sum(st_ms)) / (ms / args.steps * st_ms.size / stages),
                              "dof": dof, "roofline": roof, "launches_per_step": launches / args.steps})
            tot_dof_upd += upd
            tot_ms += ms
            tot_launch += launches

            # end to end through the public C ABI with host buffers: per step the
            # state goes host->device (pinned), one RK step runs, and the new
            # state comes back device->host.
            if args.e2e_steps > 0:
                # host buffers: the rank's compact input (owned + halo) and its owned output
                pin = torch.empty(c0.size, dtype=torch.float64, pin_memory=True)
                hbuf = pin.numpy().reshape(c0.shape)
                hbuf[...] = c0
                hp = hbuf.ctypes.data_as(L.c_double_p)
                n_out = 4 * np_(p) * N
                pout = torch.empty(n_out, dtype=torch.float64, pin_memory=True)
                op = pout.numpy().ctypes.data_as(L.c_double_p)
                # the asynchronous copy calls put each direction on its own copy stream: step
                # k+1's input is copied in (staged) while step k computes and step k's result
                # is copied out (full-duplex PCIe); the commit orders the staged input after
                # step k's download on the compute stream
                def requests(n):
                    dg2d._check(L.lib.dgb_upload_async(h, L.SLOT_STATE, hp))
                    for k in range(n):
                        if k + 1 < n:
                            dg2d._check(L.lib.dgb_stage_input_async(h, hp))
                        dg2d._check(L.lib.dgb_run_fixed_steps(h, scheme, args.cfl, 0, 1, C.byref(res), None))
                        dg2d._check(L.lib.dgb_download_async(h, L.SLOT_STATE, op))
                        if k + 1 < n:
                            dg2d._check(L.lib.dgb_commit_input(h, L.SLOT_STATE))
                    dg2d._check(L.lib.dgb_sync(h))

                requests(2)  # warm-up
                barrier(pg)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                requests(args.e2e_steps)
                ev1.record(stream)
                torch.cuda.synchronize()
                wall = (time.perf_counter() - t0) * 1e3
                ms_e = max_over_ranks(max(ev0.elapsed_time(ev1), wall), pg, local)
                e2e_dof += dof * stages * args.e2e_steps
                e2e_ms += ms_e
                h2d += c0.nbytes * world
                d2h += n_out * 8 * world
                per_order[-1]["e2e_value"] = dof * stages * args.e2e_steps / (ms_e * 1e-3)
            ctx.close()
        if world == 1 and not args.no_legs:
            for name, fn in (("c3", leg_c3), ("c4", leg_c4), ("c5", leg_c5), ("limiter_overhead", leg_limiter_overhead)):
                try:
                    legs[name] = fn(args, local, stream, hbm_gbs, fp64_tf)
                except Exception as e:  # an informational leg must never break the headline
                    legs[name] = {"failed": repr(e)}
        elif world > 1 and not args.no_legs:
            try:
                legs["c5"] = leg_c5_partitioned(args, rank, world, local, stream, pg, hbm_gbs, fp64_tf)
            except Exception as e:  # an informational leg must never break the headline
                legs["c5"] = {"failed": repr(e)}

    dom = max(per_order, key=lambda r: r["stage_kernel_ms_median"] * stages)
    line = {
        "metric": METRIC, "value": tot_dof_upd / (tot_ms * 1e-3), "unit": "DOF-updates/s/stage",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: periodic isentropic vortex initial data (projected), no dataset",
        "config": {"workload": f"isentropic vortex, periodic {n}x{n * world} box ({N_glob} triangles), "
                               f"p={','.join(map(str, orders))} sweep, {args.scheme.upper()}, cfl {args.cfl}",
                   "blend": "value = sum over the orders of the DOF updates (4 Np N x stages x K steps) / sum "
                            "over the orders of the device time of their K-step runs (each order weighs by its "
                            "own time; per-order values in per_order)",
                   "triangles_per_gpu": N, "edges_per_gpu": mesh.n_edges() // world, "orders": orders,
                   "scheme": args.scheme, "stages_per_step": stages,
                   "l2": "inputs larger than L2 (>=288 MB of coefficients per stage)",
                   "timing": "value: K steps without per-kernel events; roofline kernel_ms: median over >= 100 "
                             "stage-kernel launches timed with CUDA events on their stream in a second pass",
                   "parallelism": (f"element partition x{world} (contiguous strips), peer-memory halo "
                                   "exchange by a push kernel right behind the boundary-element stage launch") if world > 1 else "single GPU"},
        "roofline": dict(dom["roofline"], p=dom["p"],
                         note=f"dominant kernel = fused stage kernel at p={dom['p']} (median launch); "
                              f"HBM peak {hbm_src}; FP64 peak measured in-run (DFMA loop) {fp64_tf:.1f} TF/s"),
        "per_order": per_order,
        "gpu_launches": tot_launch,
        "clocks": sampler.summary(),
        "fp64_peak_tflops_measured": fp64_tf,
    }
    if e2e_ms > 0:
        line["e2e"] = {"value": e2e_dof / (e2e_ms * 1e-3), "unit": "DOF-updates/s/stage",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "note": "per step: pinned host state -> dgb_stage_input_async + dgb_commit_input -> one RK step -> dgb_download_async (one copy stream per direction: step k+1's upload overlaps step k's compute and download); wall clock incl. dgb_sync"}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(orders, args)
    line.update(legs)
    return line


def _leg_context(mesh, p, bc, opts, local, stream, c0):
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    ctx = dg2d.SolverContext(mesh, dg2d.build_tables(p), bc=bc, options=opts, device=local)
    dg2d._check(L.lib.dgb_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
    ctx.upload(L.SLOT_STATE, c0)
    return ctx


def leg_c3(args, local, stream, hbm_gbs, fp64_tf):
    """BASELINE configs[2] (C3): supersonic vortex / channel with wall BCs, p = 3, ~1M
    triangles (vortex level 6: 737,280 triangles; curved reflecting walls, Dirichlet inflow,
    outflow), SSP-RK3, cfl 0.3.  Exercises the boundary-code instance of the DMMA kernel."""
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    mesh = dg2d.generate_mesh(L.MESH_VORTEX, args.c3_level, 0, 1.0, 1.384)
    N, e = mesh.n_elements(), mesh.n_edges() / mesh.n_elements()
    c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, dg2d.build_tables(3))
    ctx = _leg_context(mesh, 3, dg2d.vortex_boundary(), dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3), local,
                       stream, c0)
    res = C.c_double()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, L.SSP_RK3, 0.3, 0, args.warmup, C.byref(res), None))
    ms, launches, st, _ = timed_run(ctx.handle, stream, L.SSP_RK3, 0.3, False, args.steps)
    ctx.close()
    k = float(np.median(st))
    upd = 4 * np_(3) * N * 3 * args.steps
    return {"workload": f"supersonic vortex level {args.c3_level} ({N} triangles, walls + inflow + outflow), p=3, "
                        "SSP-RK3, cfl 0.3", "steps": args.steps, "value": upd / (ms * 1e-3),
            "unit": "DOF-updates/s/stage", "ms_per_step": ms / args.steps, "stage_kernel_ms_median": k,
            "stage_kernel_samples": int(st.size), "roofline": roofline(3, e, N, k, hbm_gbs, fp64_tf)}


def leg_c4(args, local, stream, hbm_gbs, fp64_tf):
    """BASELINE configs[3] (C4): double Mach reflection, p = 1, Barth-Jespersen limiter on
    every stage, midpoint RK2 (dmr_desk.cfg), on the 2000x500 channel (2M triangles): the
    paper's own headline path (GTX 580 mesh C: 1.31e8 DOF-updates/s/stage)."""
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    nx, ny = args.dmr_nx, args.dmr_nx // 4
    mesh = dg2d.generate_mesh(L.MESH_DOUBLE_MACH, nx, ny, 1.0 / 6.0)
    N, e = mesh.n_elements(), mesh.n_edges() / mesh.n_elements()
    tb = dg2d.build_tables(1)
    setup = dg2d.DoubleMachSetup()
    bc = dg2d.double_mach_boundary(setup)
    opts = dg2d.SolverOptions(rk_order=2, cfl=0.3, limiting=True)
    lim = dg2d.SolverContext(mesh, tb, bc=bc, options=opts, device=local)
    c0 = dg2d.limit(lim, dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb))
    lim.close()
    ctx = _leg_context(mesh, 1, bc, opts, local, stream, c0)
    res = C.c_double()
    dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.3, 1, args.warmup, C.byref(res), None))
    # the default launch form at this size (two kernels per stage above 400K triangles: the stage
    # kernel, then the limiter kernel)
    ms, launches, st, lm = timed_run(ctx.handle, stream, 2, 0.3, True, args.steps, stages=2)
    # the same run as one fused stage + limiter launch per stage (the small-mesh default)
    L.lib.dgb_set_fused_limiter(ctx.handle, 1)
    ms_f, _, st_f, _ = timed_run(ctx.handle, stream, 2, 0.3, True, args.steps, stages=2)
    ctx.close()
    upd = 4 * 3 * N * 2 * args.steps
    k, lk, kf = float(np.median(st)), float(np.median(lm)) if lm.size else 0.0, float(np.median(st_f))
    return {"workload": f"double Mach reflection {nx}x{ny} channel ({N} triangles), p=1, BJ limiter every "
                        f"stage, RK2 midpoint, cfl 0.3", "steps": args.steps,
            "value": upd / (ms * 1e-3), "unit": "DOF-updates/s/stage", "ms_per_step": ms / args.steps,
            "launch": "stage kernel + limiter kernel per stage (the default above 400K triangles)",
            "stage_kernel_ms_median": k, "limiter_ms_median": lk, "stage_kernel_samples": int(st.size),
            "limiter_share": lk / (k + lk) if lk else None,
            "limiter_overhead": lk / k if lk else None,
            "fused": {"value": upd / (ms_f * 1e-3), "kernel_ms_median": kf,
                      "launch": "stage + limiter in one cooperative launch (k_stage_limit)"},
            "roofline_stage": roofline(1, e, N, k, hbm_gbs, fp64_tf),
            "vs_paper_gtx580_mesh_c": upd / (ms * 1e-3) / 1.31e8}


def leg_c5(args, local, stream, hbm_gbs, fp64_tf):
    """BASELINE configs[4] (C5) at N=1: the synthetic 8M-triangle box (2000 x 2000, periodic,
    isentropic vortex), p = 2..4, SSP-RK3 — the single-GPU point of the scaling curve
    (bench.py --gpus N runs the partitioned form with N x the triangles)."""
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    n = args.c5_n
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
    N, e = mesh.n_elements(), mesh.n_edges() / mesh.n_elements()
    out = {"workload": f"periodic {n}x{n} box ({N} triangles), isentropic vortex, SSP-RK3, cfl 0.3",
           "steps": args.steps, "per_order": []}
    upd_tot, ms_tot = 0.0, 0.0
    iv = dg2d.IsentropicVortex()
    for p in [int(x) for x in args.c5_orders.split(",")]:
        tb = dg2d.build_tables(p)
        ctx = dg2d.SolverContext(mesh, tb, options=dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3), device=local)
        dg2d._check(L.lib.dgb_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
        dg2d.project_on_device(ctx, iv)
        res = C.c_double()
        dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, L.SSP_RK3, 0.3, 0, args.warmup, C.byref(res), None))
        ms, launches, st, _ = timed_run(ctx.handle, stream, L.SSP_RK3, 0.3, False, args.steps)
        ctx.close()
        k = float(np.median(st))
        upd = 4 * np_(p) * N * 3 * args.steps
        upd_tot += upd
        ms_tot += ms
        out["per_order"].append({"p": p, "value": upd / (ms * 1e-3), "ms_per_step": ms / args.steps,
                                 "stage_kernel_ms_median": k, "roofline": roofline(p, e, N, k, hbm_gbs, fp64_tf)})
    out["value"] = upd_tot / (ms_tot * 1e-3)
    out["unit"] = "DOF-updates/s/stage"
    return out


def leg_c5_partitioned(args, rank, world, local, stream, pg, hbm_gbs, fp64_tf):
    """BASELINE configs[4] (C5) at N > 1: the 8M-triangle box (2000 x 2000, periodic, isentropic
    vortex), p = 2..4, SSP-RK3, partitioned across the N ranks (contiguous strips, peer-memory
    halo exchange, CUDA IPC between the processes): strong scaling of a fixed mesh, device-timed
    as the max over ranks.  The halo bytes per stage are the send lists' element columns x 4 Np
    doubles, pushed by the halo push kernel (k_push) over NVLink P2P."""
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    from paper_1601_07944_b200 import dist as D
    n = args.c5_n
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n, 10.0, 10.0)
    N, e = mesh.n_elements(), mesh.n_edges() / mesh.n_elements()
    out = {"workload": f"periodic {n}x{n} box ({N} triangles) partitioned over {world} ranks, isentropic vortex, "
                       "SSP-RK3, cfl 0.3", "scaling": "strong", "steps": args.steps, "per_order": []}
    upd_tot, ms_tot = 0.0, 0.0
    iv = dg2d.IsentropicVortex()
    for p in [int(x) for x in args.c5_orders.split(",")]:
        tb = dg2d.build_tables(p)
        ctx = D.PartContext(mesh, tb, rank, world, options=dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3),
                            device=local)
        D.connect_process_group(ctx)
        dg2d._check(L.lib.dgb_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)))
        ctx.upload(L.SLOT_STATE, D.project_local(ctx, lambda xy: iv(xy)))
        res = C.c_double()
        dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, L.SSP_RK3, 0.3, 0, args.warmup, C.byref(res), None))
        ms, launches, st, _ = timed_run(ctx.handle, stream, L.SSP_RK3, 0.3, False, args.steps, pg, local)
        info = ctx.info
        ctx.close()
        k = float(np.median(st))
        upd = 4 * np_(p) * N * 3 * args.steps
        upd_tot += upd
        ms_tot += ms
        out["per_order"].append({"p": p, "value": upd / (ms * 1e-3), "ms_per_step": ms / args.steps,
                                 "stage_kernel_ms_median_rank0": k, "owned_rank0": int(info.n_owned),
                                 "halo_rank0": int(info.n_halo),
                                 "halo_bytes_per_stage_rank0": int(info.n_halo) * 4 * np_(p) * 8,
                                 "launches_per_step": launches / args.steps,
                                 "roofline_rank0": roofline(p, e, int(info.n_owned), k, hbm_gbs, fp64_tf)})
    out["value"] = upd_tot / (ms_tot * 1e-3)
    out["unit"] = "DOF-updates/s/stage"
    out["exchange"] = "CUDA IPC peer mappings (dgb_part_attach_peer_ipc); halo columns written by the push kernel (k_push) behind the boundary stage launch"
    return out


def leg_limiter_overhead(args, local, stream, hbm_gbs, fp64_tf):
    """The reference's limiter-overhead criterion exactly as proj/tests/acceptance.cpp:368-405
    defines it: supersonic vortex mesh C (level 2), p = 1, RK2, cfl 0.9, 200 warm-up steps,
    then 10,000 steps timed with limiting off and on (the "on" run starts from the limited
    projection); overhead = (t_on - t_off) / t_off (threshold 25%, PAPER.md:1060 <= 15%)."""
    import torch
    from paper_1601_07944_b200 import _lib as L
    from paper_1601_07944_b200 import dg2d
    mesh = dg2d.generate_mesh(L.MESH_VORTEX, 2, 0, 1.0, 1.384)
    tb = dg2d.build_tables(1)
    c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, tb)
    times = {}
    for lim in (False, True):
        opts = dg2d.SolverOptions(rk_order=2, cfl=0.9, limiting=lim)
        ctx = _leg_context(mesh, 1, dg2d.vortex_boundary(), opts, local, stream, c0)
        if lim:
            ctx.upload(L.SLOT_STATE, dg2d.limit(ctx, c0.copy()))
        res = C.c_double()
        dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.9, int(lim), 200, C.byref(res), None))
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        dg2d._check(L.lib.dgb_run_fixed_steps(ctx.handle, 2, 0.9, int(lim), args.lim_steps, C.byref(res), None))
        ev1.record(stream)
        torch.cuda.synchronize()
        times["on" if lim else "off"] = ev0.elapsed_time(ev1)
        ctx.close()
    return {"workload": f"supersonic vortex mesh C (level 2, {mesh.n_elements()} triangles), p=1, RK2, cfl 0.9, "
                        f"{args.lim_steps} steps after 200 warm-up (acceptance.cpp:368-405)",
            "ms_off": times["off"], "ms_on": times["on"],
            "overhead": (times["on"] - times["off"]) / times["off"], "threshold": 0.25}


# ----------------------------------------------------------------------------- CPU reference
REF_CONFIG_NOTE = ("same mesh (the periodic 708x708 box built by the reference's own build_connectivity with "
                   "the hull edges joined, array-identical to ours: tests/test_host_setup.py), same initial data "
                   "(the reference's project_initial of the same isentropic vortex), same orders; the reference "
                   "has no SSP-RK3, so it runs its RK2 midpoint scheme: a stage is one compute_rhs + the stage "
                   "combination in both, and the metric is per stage")


def cpu_sample(orders, n, steps=2):
    """The reference solver (oracle/_ref, -march=native, OpenMP over every host core, bound
    close) on the benchmark's own workload: one run_fixed_steps call of `steps` RK2 steps
    per order.  Returns the cpu_baseline object."""
    from oracle import refarm
    if not refarm.available():
        raise RuntimeError("oracle/_ref not built")
    r = refarm.throughput(n, orders, calls_per_order=1, steps_per_call=steps, warmup_calls=0)
    secs = sum(r["best_s"].values())
    return {"value": r["value"], "unit": "DOF-updates/s/stage", "cores": r["threads"], "kind": "reference",
            "seconds": secs, "library": r["so"],
            "sample": f"one run_fixed_steps call of {steps} RK2 (midpoint) steps per order "
                      f"p={','.join(map(str, orders))} on the periodic {n}^2 box ({r['N']} triangles), the "
                      f"reference's own build (-O3 -march=native -fno-math-errno, OpenMP over {r['threads']} "
                      "threads, unbound: the reference runs its own worker pool), no warm-up"}


def cpu_baseline(orders, args):
    try:
        return cpu_sample(orders, args.cpu_n)
    except Exception as e:  # the CPU leg must never break the GPU number
        return {"value": None, "unit": "DOF-updates/s/stage", "cores": None, "kind": None,
                "sample": f"failed: {e}"}


def run_reference(args, rank, world):
    """The reference arm: the UNMODIFIED reference's CPU solver (oracle/refarm.py; this
    process never loads the B200 library).  A bench step is one run_fixed_steps call of
    --ref-steps RK2 steps (the reference's own driver, its RkWorkspace reused across the
    steps of the call, solver.cpp:600-613) at one order, the orders taken round robin; after
    one untimed warm-up call per order.  value = sum over orders of the DOF updates of one call
    / sum of each order's best timed call (best of >= 3 when --steps >= 3 x orders)."""
    if rank != 0:
        return None
    from oracle import refarm
    orders = [int(x) for x in args.orders.split(",")]
    sched = [orders[k % len(orders)] for k in range(args.steps)]
    warm = max(1, -(-args.warmup // len(orders)))
    r = refarm.throughput(args.cpu_n, orders, calls_per_order=0, steps_per_call=args.ref_steps,
                          warmup_calls=warm, schedule=sched)
    value, N = r["value"], r["N"]
    t_tot = sum(sum(v) for v in r["all_s"].values())
    sample = (f"one run_fixed_steps call of {args.ref_steps} RK2 (midpoint) steps per bench step, orders "
              f"p={args.orders} round robin, on the periodic {args.cpu_n}^2 box ({N} triangles); per order the best "
              f"of its {min(len(v) for v in r['all_s'].values())}+ timed calls; the reference's own build "
              f"({r['so']}: -O3 -march=native -fno-math-errno) with OpenMP over {r['threads']} threads, "
              "unbound (the reference runs its own worker pool))")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF-updates/s/stage",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_tot / max(len(sched), 1) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic: periodic isentropic vortex initial data (projected)",
        "config": {"workload": f"isentropic vortex, periodic {args.cpu_n}x{args.cpu_n} box ({N} triangles), "
                               f"p={args.orders} sweep, reference RK2 midpoint, cfl 0.3",
                   "orders": orders, "same_config": REF_CONFIG_NOTE},
        "per_order": {str(p): v for p, v in r["per_order"].items()},
        "cpu_baseline": {"value": value, "unit": "DOF-updates/s/stage", "cores": r["threads"],
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "DOF-updates/s/stage", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--box", dest="n", type=int, default=708, help="box cells per side (2 n^2 triangles per GPU)")
    ap.add_argument("--orders", default="1,2,3,4,5")
    ap.add_argument("--scheme", default="ssp3", choices=list(SCHEMES))
    ap.add_argument("--cfl", type=float, default=0.3)
    ap.add_argument("--e2e-steps", type=int, default=32, help="requests per order in the end-to-end leg (the pipeline fills and drains once)")
    ap.add_argument("--cpu-box", dest="cpu_n", type=int, default=708, help="box size of the CPU sample")
    ap.add_argument("--ref-steps", type=int, default=3, help="RK2 steps per reference run_fixed_steps call")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dmr-nx", type=int, default=2000, help="DMR channel cells in x (C4 leg)")
    ap.add_argument("--c3-level", type=int, default=6, help="supersonic-vortex mesh level of the C3 leg")
    ap.add_argument("--c5-n", type=int, default=2000, help="box cells per side of the C5 leg (2 n^2 triangles)")
    ap.add_argument("--c5-orders", default="2,3,4")
    ap.add_argument("--lim-steps", type=int, default=10000, help="steps of the limiter-overhead leg")
    ap.add_argument("--no-legs", action="store_true", help="headline sweep only (no C3/C4/C5/limiter legs)")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: all ranks share cuda:0 (partitioned path on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        # the reference arm is CPU-only: rank 0 runs it, the other ranks exit at once, and no
        # rank touches CUDA or a process group
        rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
        line, pg = run_reference(args, rank, world), None
    else:
        rank, world, local, pg = dist_setup(args.gpus, args.same_device)
        line = run_b200(args, rank, world, local, pg)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
