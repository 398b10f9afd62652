"""Multi-GPU element partition with a peer-memory halo exchange.

Rank r of ``world`` owns the contiguous reference ids ``[n*r/world, n*(r+1)/world)``.  Its
device context (``dgb_part_create``) holds the owned elements plus halo columns for the
off-rank neighbours.  Every RK stage the stage kernel itself writes the elements a peer needs
into that peer's halo columns (peer memory over NVLink), then raises an epoch flag; each
rank computes its interior elements while the peers' halo data is in flight.  The global
CFL bound, residual and error key are merged the same way once per step.  There is no NCCL
on the data path: ``torch.distributed`` (any backend) only carries the CUDA IPC handles and
the halo id lists at setup.

Two ways to wire the ranks:

* ``connect_local(parts)`` — several partitions in ONE process (same or different devices),
  attached with raw device pointers; ``run_group`` drives them from one thread each
  (ctypes releases the GIL).  This is how the partitioned path is tested on a single GPU.
* ``connect_process_group(part)`` — one process per GPU (``torchrun``), attached through
  CUDA IPC handles exchanged with ``torch.distributed.all_gather_object``.

Coefficient arrays cross the ABI in "compact" order: owned ids then halo ids
(``local_ids``).  ``PartContext.upload`` takes compact arrays only and
``PartContext.upload_global`` takes a reference-layout global array (it gathers the
rank's columns); the shapes are checked, never guessed.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Callable, List, Sequence

import numpy as np

from . import _lib as L
from ._lib import dptr, iptr, lib
from .dg2d import SolverContext, SolverState, _check, kEq


def plan(mesh, rank: int, world: int) -> dict:
    """Host-only partition plan (no device): owned range, halo ids, boundary ids."""
    info = L.PartInfo()
    _check(lib.dgb_part_plan(C.byref(mesh.view), rank, world, C.byref(info), None, None))
    halo = np.zeros(max(info.n_halo, 1), np.int32)
    bnd = np.zeros(max(info.n_owned - info.n_interior, 1), np.int32)
    _check(lib.dgb_part_plan(C.byref(mesh.view), rank, world, C.byref(info), iptr(halo), iptr(bnd)))
    return {"rank": rank, "world": world, "lo": info.lo, "hi": info.hi, "n_owned": info.n_owned,
            "n_halo": info.n_halo, "n_interior": info.n_interior, "ld": info.ld,
            "neighbor_mask": info.neighbor_mask, "halo_ids": halo[:info.n_halo],
            "halo_cols": np.arange(info.n_owned, info.n_owned + info.n_halo, dtype=np.int32),
            "boundary_ids": bnd[:info.n_owned - info.n_interior]}


def owner_of(ids, n: int, world: int) -> np.ndarray:
    """Rank owning each reference id under the contiguous partition."""
    ids = np.asarray(ids, np.int64)
    r = (ids * world) // n
    lo = (r * n) // world
    r = np.where(ids < lo, r - 1, r)
    hi = ((r + 1) * n) // world
    return np.where(ids >= hi, r + 1, r).astype(np.int64)


def send_lists(plans: Sequence[dict], sender: int, n: int) -> dict:
    """For rank ``sender``: {peer: (ids owned by sender that peer holds as halo, peer columns)}."""
    out = {}
    for p in plans:
        if p["rank"] == sender:
            continue
        own = owner_of(p["halo_ids"], n, p["world"]) == sender
        if own.any():
            out[p["rank"]] = (np.ascontiguousarray(p["halo_ids"][own], np.int32),
                              np.ascontiguousarray(p["halo_cols"][own], np.int32))
    return out


class PartContext(SolverContext):
    """A partition of the mesh on one device; the solver calls of ``dg2d`` work on it
    through the ordinary C ABI (dgb_run_* etc.) once the ranks are connected."""

    def __init__(self, mesh, tables, rank: int, world: int, gas=None, bc=None, options=None, device=None):
        super().__init__(mesh, tables, gas, bc, options, device)
        self.rank, self.world = rank, world
        v = self._bc_view()
        h = C.c_void_p()
        _check(lib.dgb_part_create(C.byref(mesh.view), C.byref(tables.view), C.byref(v), self.gas.gamma,
                                   self.device, rank, world, C.byref(h)))
        self._ctx = h
        lib.dgb_enable_timers(h, 1)
        _check(lib.dgb_set_flux(h, self.options.flux_id()))
        info = L.PartInfo()
        _check(lib.dgb_part_get_info(h, C.byref(info)))
        self.info = info
        nl = info.n_owned + info.n_halo
        self.local_ids = np.zeros(max(nl, 1), np.int32)
        _check(lib.dgb_part_local_ids(h, iptr(self.local_ids)))
        self.local_ids = self.local_ids[:nl]
        self.halo_ids = self.local_ids[info.n_owned:]
        self.halo_cols = np.arange(info.n_owned, nl, dtype=np.int32)
        self.owned = slice(info.lo, info.hi)

    # compact-order transfers ---------------------------------------------------------
    def _shape(self):
        return (kEq, self.tables.n_p, self.info.n_owned + self.info.n_halo)

    def upload(self, slot, coeffs):
        """Compact-order array [4][n_p][n_owned + n_halo] (owned ids, then halo ids)."""
        c = np.asarray(coeffs, np.float64)
        if c.shape != self._shape():
            raise ValueError(f"PartContext.upload takes a compact array of shape {self._shape()}, got {c.shape} "
                             "(use upload_global for a reference-layout global array)")
        super().upload(slot, np.ascontiguousarray(c))

    def upload_global(self, slot, coeffs):
        """Reference-layout global array [4][n_p][n_elements]: the rank's owned and halo
        columns are gathered in compact order."""
        c = np.asarray(coeffs, np.float64)
        if c.shape != (kEq, self.tables.n_p, self.mesh.n_elements()):
            raise ValueError(f"PartContext.upload_global takes a global array of shape "
                             f"{(kEq, self.tables.n_p, self.mesh.n_elements())}, got {c.shape}")
        self.upload(slot, c[:, :, self.local_ids])

    def download(self, slot):
        out = np.empty((kEq, self.tables.n_p, self.info.n_owned))
        _check(lib.dgb_download(self.handle, slot, dptr(out)))
        return out

    def peer_view(self) -> L.PeerView:
        v = L.PeerView()
        _check(lib.dgb_part_peer_view(self.handle, C.byref(v)))
        return v

    def ipc_handles(self) -> bytes:
        buf = (C.c_char * L.IPC_BYTES)()
        _check(lib.dgb_part_ipc_export(self.handle, buf))
        return bytes(buf)

    def set_sends(self, peer: int, ids, cols):
        ids = np.ascontiguousarray(ids, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        _check(lib.dgb_part_set_sends(self.handle, peer, ids.size, iptr(ids), iptr(cols)))

    def finalize(self):
        _check(lib.dgb_part_finalize(self.handle))

    def set_timeout(self, seconds: float):
        _check(lib.dgb_part_set_timeout(self.handle, seconds))

    def partial_mass(self, slot=L.SLOT_STATE) -> float:
        m = C.c_double()
        _check(lib.dgb_total_mass(self.handle, slot, C.byref(m)))
        return m.value


def project_local(part: "PartContext", u0: Callable) -> np.ndarray:
    """project_initial (solver.cpp:74-97) of the rank's owned + halo elements only, in
    compact order — so no rank ever materialises the global coefficient array."""
    mesh, tb = part.mesh, part.tables
    ev = np.ascontiguousarray(mesh.elem_v[part.local_ids].reshape(-1), np.int32)
    v = L.MeshView.from_buffer_copy(mesh.view)
    v.n_elements = int(part.local_ids.size)
    v.elem_v = iptr(ev)
    nl, nq = part.local_ids.size, tb.n_quad
    xy = np.empty((nl, nq, 2))
    _check(lib.dgb_interior_points(C.byref(v), C.byref(tb.view), dptr(xy)))
    vals = np.ascontiguousarray(np.asarray(u0(xy.reshape(-1, 2)), np.float64).reshape(nl, nq, 4))
    out = np.empty((kEq, tb.n_p, nl))
    _check(lib.dgb_project(C.byref(v), C.byref(tb.view), part.gas.gamma, dptr(vals), dptr(out)))
    return out


def _my_plan(part: PartContext) -> dict:
    i = part.info
    return {"rank": part.rank, "world": part.world, "lo": i.lo, "hi": i.hi, "halo_ids": part.halo_ids,
            "halo_cols": part.halo_cols}


def connect_local(parts: List[PartContext]):
    """Wire partitions living in this process (raw device pointers)."""
    views = [p.peer_view() for p in parts]
    plans = [_my_plan(p) for p in parts]
    n = parts[0].mesh.n_elements()
    for p in parts:
        for q in parts:
            if q is not p:
                _check(lib.dgb_part_attach_peer(p.handle, q.rank, C.byref(views[q.rank])))
        for peer, (ids, cols) in send_lists(plans, p.rank, n).items():
            p.set_sends(peer, ids, cols)
    for p in parts:
        p.finalize()


def connect_process_group(part: PartContext, group=None):
    """Wire one partition per process: IPC handles + halo lists via torch.distributed."""
    import torch.distributed as dist
    mine = {"rank": part.rank, "ipc": part.ipc_handles(), "ld": part.info.ld, "plan": _my_plan(part)}
    allp = [None] * part.world
    dist.all_gather_object(allp, mine, group=group)
    for o in allp:
        if o["rank"] != part.rank:
            buf = C.create_string_buffer(o["ipc"], L.IPC_BYTES)
            _check(lib.dgb_part_attach_peer_ipc(part.handle, o["rank"], buf, o["ld"]))
    plans = [o["plan"] for o in allp]
    for peer, (ids, cols) in send_lists(plans, part.rank, part.mesh.n_elements()).items():
        part.set_sends(peer, ids, cols)
    part.finalize()
    dist.barrier(group=group)


def run_group(parts: Sequence, fn: Callable):
    """Run ``fn(part)`` for every in-process partition concurrently (one host thread each);
    re-raises the first failure."""
    errs = [None] * len(parts)
    res = [None] * len(parts)

    def work(i):
        try:
            res[i] = fn(parts[i])
        except BaseException as e:  # noqa: BLE001 — re-raised below
            errs[i] = e
    th = [threading.Thread(target=work, args=(i,)) for i in range(len(parts))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return res


def run_fixed_steps_group(parts: Sequence[PartContext], state: SolverState, n_steps: int) -> float:
    """run_fixed_steps over an in-process partition group; gathers the owned results back
    into ``state`` (reference layout) and returns the global residual."""
    if any(p.bc.time_dependent and p.bc.dirichlet is not None for p in parts):
        # the device step loop of a partition group keeps one Dirichlet table per run; the
        # stage-time tables of dg2d's host-stepped drivers need a host dt, i.e. a host min over ranks
        raise ValueError("time-dependent Dirichlet data are not supported by partitioned runs "
                         "(use a whole-mesh context: dg2d.run_fixed_steps steps them on the host)")
    for p in parts:
        p.upload_global(L.SLOT_STATE, state.coeffs)
        _check(lib.dgb_set_time(p.handle, state.t, state.step_count))

    def go(p):
        r = C.c_double()
        _check(lib.dgb_run_fixed_steps(p.handle, p.options.scheme_id(), p.options.cfl, int(p.options.limiting),
                                       int(n_steps), C.byref(r), None))
        return r.value
    res = run_group(parts, go)
    out = np.array(state.coeffs, copy=True)
    for p in parts:
        out[:, :, p.owned] = p.download(L.SLOT_STATE)
    t, s = C.c_double(), C.c_int64()
    _check(lib.dgb_get_time(parts[0].handle, C.byref(t), C.byref(s)))
    state.coeffs, state.t, state.step_count = out, t.value, s.value
    return max(res)
