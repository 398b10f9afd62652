"""Multi-GPU partition: host plan checked across gloo processes on CPU, and the
peer-memory halo exchange checked on one GPU against the whole-mesh solve (bit-identical).

The GPU tests run 2-4 partitions of one mesh on cuda:0 — in one process (raw device pointers,
one host thread per partition) and in two processes (CUDA IPC handles over torch.distributed)
— so the exact kernels, flags and waits of an 8-GPU run are exercised on the single B200.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1601_07944_b200 import _lib as L
from paper_1601_07944_b200 import dg2d, dist as D



def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _neighbours(mesh):
    """[N][3] neighbour id per side (negative = boundary code), from the edge arrays."""
    e = mesh.elem_edge
    ids = np.arange(mesh.n_elements())[:, None]
    left = mesh.edge_left[e]
    right = mesh.edge_right[e]
    return np.where(left == ids, right, left)


MESHES = {
    "periodic": lambda: dg2d.generate_mesh(L.MESH_PERIODIC_BOX, 12, 9, 10.0, 10.0),
    "dmr": lambda: dg2d.generate_mesh(L.MESH_DOUBLE_MACH, 24, 6, 1.0 / 6.0),
    "vortex": lambda: dg2d.generate_mesh(L.MESH_VORTEX, 1, 0, 1.0, 1.384),
}


# ----------------------------------------------------------------------------- CPU: the plan
@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_plan_covers_mesh_and_halo_is_exact(name, world):
    mesh = MESHES[name]()
    n = mesh.n_elements()
    nb = _neighbours(mesh)
    plans = [D.plan(mesh, r, world) for r in range(world)]
    owned = np.concatenate([np.arange(p["lo"], p["hi"]) for p in plans])
    assert np.array_equal(owned, np.arange(n))  # contiguous, disjoint, complete
    for p in plans:
        mine = np.arange(p["lo"], p["hi"])
        nbs = nb[mine]
        off = (nbs >= 0) & ((nbs < p["lo"]) | (nbs >= p["hi"]))
        assert np.array_equal(np.unique(nbs[off]), p["halo_ids"])
        assert np.array_equal(np.sort(mine[off.any(1)]), p["boundary_ids"])
        assert p["n_interior"] == p["n_owned"] - p["boundary_ids"].size
        assert p["ld"] % 32 == 0 and p["ld"] >= p["n_owned"] + p["n_halo"]
        owners = set(D.owner_of(p["halo_ids"], n, world).tolist())
        assert sum(1 << r for r in owners) == p["neighbor_mask"]
        assert p["rank"] not in owners
    for r in range(world):  # sends = the peers' halo elements owned by r, all on r's boundary
        for peer, (ids, cols) in D.send_lists(plans, r, n).items():
            assert np.all((ids >= plans[r]["lo"]) & (ids < plans[r]["hi"]))
            assert np.isin(ids, plans[r]["boundary_ids"]).all()
            assert np.all(cols >= plans[peer]["n_owned"])
            assert (plans[peer]["neighbor_mask"] >> r) & 1


def _gloo_worker(rank, world, port, name, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mesh = MESHES[name]()
        n = mesh.n_elements()
        p = D.plan(mesh, rank, world)
        plans = [None] * world
        dist.all_gather_object(plans, p)
        # emulate one halo exchange with the plan: owned columns hold f(id), halo columns
        # are filled only through the send lists, over the process group
        f = lambda ids: np.sin(0.37 * np.asarray(ids, np.float64)) + ids  # noqa: E731
        local = np.full(p["n_owned"] + p["n_halo"], np.nan)
        local[:p["n_owned"]] = f(np.arange(p["lo"], p["hi"]))
        sends = D.send_lists(plans, rank, n)
        recvs = {r: D.send_lists(plans, r, n).get(rank) for r in range(world) if r != rank}
        ops = []
        for peer, (ids, cols) in sends.items():
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(local[ids - p["lo"]].copy()), peer))
        bufs = {}
        for r, sl in recvs.items():
            if sl is not None:
                bufs[r] = torch.empty(sl[0].size, dtype=torch.float64)
                ops.append(dist.P2POp(dist.irecv, bufs[r], r))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for r, b in bufs.items():
            local[recvs[r][1]] = b.numpy()
        ok = np.array_equal(local[p["n_owned"]:], f(p["halo_ids"])) and not np.isnan(local).any()
        # every rank agrees on who neighbours whom
        masks = [None] * world
        dist.all_gather_object(masks, p["neighbor_mask"])
        sym = all(((masks[a] >> b) & 1) == ((masks[b] >> a) & 1) for a in range(world) for b in range(world))
        dist.destroy_process_group()
        q.put((rank, bool(ok and sym), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("world,name", [(2, "periodic"), (2, "dmr"), (3, "periodic"), (3, "vortex")])
def test_halo_plan_exchange_over_gloo(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in out), out


# ----------------------------------------------------------------------------- GPU
def _problem(name, p):
    mesh = MESHES[name]()
    tb = dg2d.build_tables(p)
    if name == "dmr":
        setup = dg2d.DoubleMachSetup()
        bc = dg2d.double_mach_boundary(setup)
        c0 = dg2d.project_initial(lambda xy: dg2d.double_mach_initial(xy, setup), mesh, tb)
        lim = dg2d.SolverContext(mesh, tb, bc=bc, device=0)  # runner.cpp:177 limits the projection
        c0 = dg2d.limit(lim, c0)
        lim.close()
    elif name == "vortex":
        bc = dg2d.vortex_boundary()
        c0 = dg2d.project_initial(lambda xy: dg2d.vortex_exact(xy), mesh, tb)
    else:
        bc = None
        c0 = dg2d.project_initial(dg2d.IsentropicVortex(xc=5.0, yc=5.0), mesh, tb)
    return mesh, tb, bc, c0


def _whole(mesh, tb, bc, c0, opts, steps, t0=0.0, step0=0):
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts, device=0)
    st = dg2d.SolverState(c0.copy(), t0, step0)
    res = dg2d.run_fixed_steps(ctx, st, steps)
    ctx.close()
    return st, res


@pytest.mark.gpu
@pytest.mark.parametrize("name,p,scheme,world,limiting", [
    ("periodic", 1, L.SSP_RK3, 2, False), ("periodic", 2, L.RK4_CLASSIC, 3, False),
    ("periodic", 3, L.SSP_RK2, 4, False), ("periodic", 5, L.SSP_RK3, 2, False),
    ("vortex", 4, L.RK2_MIDPOINT, 3, False), ("dmr", 1, L.RK2_MIDPOINT, 3, True),
    ("dmr", 1, L.SSP_RK3, 2, True)])
def test_in_process_partitions_bit_identical_to_whole_mesh(name, p, scheme, world, limiting):
    mesh, tb, bc, c0 = _problem(name, p)
    opts = dg2d.SolverOptions(scheme=scheme, cfl=0.3, limiting=limiting)
    steps = 12
    ref, res_ref = _whole(mesh, tb, bc, c0, opts, steps)
    parts = [D.PartContext(mesh, tb, r, world, bc=bc, options=opts, device=0) for r in range(world)]
    for q in parts:
        q.set_timeout(30.0)
    D.connect_local(parts)
    st = dg2d.SolverState(c0.copy())
    res = D.run_fixed_steps_group(parts, st, steps)
    assert np.array_equal(st.coeffs, ref.coeffs), np.max(np.abs(st.coeffs - ref.coeffs))
    assert st.t == ref.t and st.step_count == ref.step_count
    assert res == res_ref
    # a second call continues the same epoch sequence
    ref2, _ = _whole(mesh, tb, bc, ref.coeffs, opts, 3, ref.t, ref.step_count)
    D.run_fixed_steps_group(parts, st, 3)
    assert np.array_equal(st.coeffs, ref2.coeffs) and st.t == ref2.t
    mass = sum(q.partial_mass() for q in parts)
    assert abs(mass - dg2d.total_mass(mesh, st.coeffs)) <= 1e-12 * abs(mass)
    for q in parts:
        q.close()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs in this process")
@pytest.mark.parametrize("p,limiting", [(1, True), (3, False), (5, False)])
def test_partitions_on_different_devices_bit_identical(p, limiting):
    """connect_local across devices: dgb_part_attach_peer enables P2P access between the
    devices, and the halo stores cross NVLink; bit-identical to the whole-mesh solve."""
    ndev = min(torch.cuda.device_count(), 4)
    name = "dmr" if limiting else "periodic"
    mesh, tb, bc, c0 = _problem(name, p)
    opts = dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3, limiting=limiting)
    ref, res_ref = _whole(mesh, tb, bc, c0, opts, 10)
    parts = [D.PartContext(mesh, tb, r, ndev, bc=bc, options=opts, device=r) for r in range(ndev)]
    for q in parts:
        q.set_timeout(30.0)
    D.connect_local(parts)
    st = dg2d.SolverState(c0.copy())
    res = D.run_fixed_steps_group(parts, st, 10)
    assert np.array_equal(st.coeffs, ref.coeffs)
    assert res == res_ref and st.t == ref.t
    for q in parts:
        q.close()


@pytest.mark.gpu
def test_partition_upload_layout_is_explicit():
    """upload takes compact arrays only, upload_global reference-layout ones (a
    shape guess passes a global array through unpermuted whenever n_owned + n_halo equals
    n_elements, e.g. rank 1 of the two-element mesh, whose compact order is [1, 0])."""
    mesh, tb, bc, c0 = _problem("periodic", 1)
    parts = [D.PartContext(mesh, tb, r, 2, device=0) for r in range(2)]
    q = parts[1]
    with pytest.raises(ValueError):
        q.upload(L.SLOT_STATE, c0)  # global array through the compact entry
    q.upload_global(L.SLOT_STATE, c0)
    q.upload(L.SLOT_STATE, c0[:, :, q.local_ids])
    for r in parts:
        r.close()


@pytest.mark.gpu
def test_partition_run_to_time_halts_together():
    mesh, tb, bc, c0 = _problem("periodic", 2)
    opts = dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3)
    ctx = dg2d.SolverContext(mesh, tb, options=opts, device=0)
    ref = dg2d.SolverState(c0.copy())
    dg2d.run_to_time(ctx, ref, 0.05, 10_000)
    parts = [D.PartContext(mesh, tb, r, 3, options=opts, device=0) for r in range(3)]
    D.connect_local(parts)
    for q in parts:
        q.upload_global(L.SLOT_STATE, c0)

    def go(q):
        import ctypes as C
        r, n = C.c_double(), C.c_int64()
        dg2d._check(L.lib.dgb_run_to_time(q.handle, L.SSP_RK3, 0.3, 0, 0.05, 10_000, C.byref(r), C.byref(n), None, 0))
        return n.value
    steps = D.run_group(parts, go)
    assert len(set(steps)) == 1 and steps[0] == ref.step_count
    out = np.empty_like(c0)
    for q in parts:
        out[:, :, q.owned] = q.download(L.SLOT_STATE)
    assert np.array_equal(out, ref.coeffs)


def _ipc_worker(rank, world, port, q, p=3):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mesh, tb, bc, c0 = _problem("periodic", p)
        opts = dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3)
        part = D.PartContext(mesh, tb, rank, world, options=opts, device=0)
        part.set_timeout(60.0)
        D.connect_process_group(part)
        st = dg2d.SolverState(c0.copy())
        part.upload_global(L.SLOT_STATE, st.coeffs)
        import ctypes as C
        r = C.c_double()
        dg2d._check(L.lib.dgb_run_fixed_steps(part.handle, L.SSP_RK3, 0.3, 0, 6, C.byref(r), None))
        mine = part.download(L.SLOT_STATE)
        allp = [None] * world
        dist.all_gather_object(allp, (part.info.lo, part.info.hi, mine))
        dist.barrier()
        part.close()
        dist.destroy_process_group()
        if rank == 0:
            out = np.empty_like(c0)
            for lo, hi, a in allp:
                out[:, :, lo:hi] = a
            q.put((rank, out, r.value, ""))
        else:
            q.put((rank, None, r.value, ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, None, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("p", [3, 5])  # p = 5: the trace rows travel with the coefficient rows
def test_two_processes_ipc_halo_exchange_bit_identical(p):
    mesh, tb, bc, c0 = _problem("periodic", p)
    opts = dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3)
    ref, res_ref = _whole(mesh, tb, bc, c0, opts, 6)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, p)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
    assert all(o[3] == "" for o in out), out
    assert np.array_equal(out[0][1], ref.coeffs)
    assert out[0][2] == res_ref and out[1][2] == res_ref


@pytest.mark.gpu
def test_eight_partitions_roe_flux_bit_identical():
    """kMaxRanks = 8 partitions of one mesh (the 8xB200 box) with the Roe flux, in one process."""
    mesh, tb, bc, c0 = _problem("periodic", 3)
    opts = dg2d.SolverOptions(scheme=L.SSP_RK3, cfl=0.3, flux="roe")
    ref, res_ref = _whole(mesh, tb, bc, c0, opts, 6)
    parts = [D.PartContext(mesh, tb, r, 8, options=opts, device=0) for r in range(8)]
    for q in parts:
        q.set_timeout(30.0)
    D.connect_local(parts)
    st = dg2d.SolverState(c0.copy())
    res = D.run_fixed_steps_group(parts, st, 6)
    assert np.array_equal(st.coeffs, ref.coeffs) and res == res_ref
    for q in parts:
        q.close()


@pytest.mark.gpu
def test_partition_run_to_steady_matches_whole_mesh():
    """run_to_steady (solver.cpp:559-579) on the supersonic vortex, 3 partitions: the global
    residual decides the stop, so every rank takes the same number of steps."""
    mesh, tb, bc, c0 = _problem("vortex", 2)
    opts = dg2d.SolverOptions(rk_order=4, cfl=0.9)
    ctx = dg2d.SolverContext(mesh, tb, bc=bc, options=opts, device=0)
    ref = dg2d.SolverState(c0.copy())
    sr = dg2d.run_to_steady(ctx, ref, 1e-9, 20_000)
    assert sr.converged
    parts = [D.PartContext(mesh, tb, r, 3, bc=bc, options=opts, device=0) for r in range(3)]
    D.connect_local(parts)
    for q in parts:
        q.upload_global(L.SLOT_STATE, c0)

    def go(q):
        import ctypes as C
        n, r, conv = C.c_int64(), C.c_double(), C.c_int()
        dg2d._check(L.lib.dgb_run_to_steady(q.handle, 4, 0.9, 0, 1e-9, 20_000, C.byref(n), C.byref(r),
                                            C.byref(conv), None, 0))
        return n.value, r.value, conv.value
    outs = D.run_group(parts, go)
    assert all(o == (sr.steps, sr.residual, 1) for o in outs), (outs, sr)
    out = np.empty_like(c0)
    for q in parts:
        out[:, :, q.owned] = q.download(L.SLOT_STATE)
    assert np.array_equal(out, ref.coeffs)


def test_plan_rejects_bad_arguments():
    mesh = MESHES["periodic"]()
    for rank, world in ((0, 0), (0, 9), (2, 2), (-1, 2)):
        with pytest.raises(ValueError):
            D.plan(mesh, rank, world)
    tiny = dg2d.generate_mesh(L.MESH_BOX, 1, 1, 1.0, 1.0, 4)  # 2 triangles
    with pytest.raises(ValueError):
        D.plan(tiny, 0, 3)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_strip_partition_of_the_bench_box_has_two_neighbours(world):
    """The bench's weak-scaling box (n x n*world cells, periodic): every rank owns exactly
    2 n^2 triangles and exchanges halos with its two strip neighbours only."""
    n = 12
    mesh = dg2d.generate_mesh(L.MESH_PERIODIC_BOX, n, n * world, 10.0, 10.0 * world)
    for r in range(world):
        p = D.plan(mesh, r, world)
        assert p["n_owned"] == 2 * n * n
        nbrs = {k for k in range(world) if (p["neighbor_mask"] >> k) & 1}
        assert nbrs == {(r - 1) % world, (r + 1) % world}
        assert p["n_halo"] <= 4 * n  # one row of cells above and below
