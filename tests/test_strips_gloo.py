"""Row-strip decomposition host logic, including a world_size-2 gloo run of the halo protocol.

The device path exchanges the same contiguous row ranges with NCCL; here the protocol is run on
CPU tensors with torch.distributed (gloo) to check that after one exchange every ghost row holds
its owner's values and that all-reducing owned partial sums reproduces the global sums.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_07969_b200 import meshing, strips

MESHES = {
    "notched16": lambda: meshing.build_notched_square(16, 16, 1.0),
    "notched64": lambda: meshing.build_notched_square(64, 64, 1.0),
    "lshape": lambda: meshing.build_lshape_mesh(12.5),
    "plain32": lambda: meshing.build_notched_square(32, 32, 1000.0, False),
}


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_strips_partition_the_mesh(name, nranks):
    mesh = MESHES[name]()
    lay = meshing.StructuredLayout.from_mesh(mesh)
    try:
        cuts = strips.partition_rows(lay, nranks)
    except ValueError:
        assert lay.ny + 1 < 3 * nranks  # only tiny meshes may be uncuttable
        pytest.skip("too few node rows for this many strips around the slit")
    nodes, cells = [], []
    for r in range(nranks):
        st = strips.make_strip(lay, nranks, r, cuts)
        lc = st.layout.connectivity()
        assert np.array_equal(st.local_to_global[lc], mesh.elements[st.cell_local_to_global])
        nodes.append(st.owned_global_nodes())
        cells.append(st.cell_local_to_global[st.cell_lo:st.cell_hi])
        if lay.notch_row >= 0:
            assert st.jlo != lay.notch_row + 1  # never needs the duplicates as ghosts
    assert np.array_equal(np.sort(np.concatenate(nodes)), np.arange(mesh.n_nodes))
    assert np.array_equal(np.sort(np.concatenate(cells)), np.arange(mesh.n_elems))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = MESHES[name]()
        lay = meshing.StructuredLayout.from_mesh(mesh)
        st = strips.make_strip(lay, world, rank)
        rng = np.random.default_rng(5)
        u_glob = rng.standard_normal((mesh.n_nodes, 2))
        u_loc = u_glob[st.local_to_global].copy()
        ghost = np.ones(st.n_local, bool)
        ghost[st.own_lo:st.own_hi] = False
        ghost[st.dup_lo:] = False
        u_loc[ghost] = np.nan  # ghosts start invalid

        def send(dst, arr):
            dist.send(torch.from_numpy(np.ascontiguousarray(arr).ravel()), dst)

        def recv(src, n):
            t = torch.empty(n, dtype=torch.float64)
            dist.recv(t, src)
            return t.numpy()

        # even ranks send first, odd ranks receive first (blocking gloo point-to-point)
        if rank % 2 == 0:
            strips.halo_exchange(st, u_loc, 2, send, recv)
        else:
            v = u_loc.reshape(-1, 2)
            for side in ("lo", "hi"):
                rr = getattr(st, f"recv_{side}")
                if rr is not None:
                    s, n = rr
                    v[s:s + n] = recv(rank - 1 if side == "lo" else rank + 1, 2 * n).reshape(n, 2)
            for side in ("lo", "hi"):
                ss = getattr(st, f"send_{side}")
                if ss is not None:
                    s, n = ss
                    send(rank - 1 if side == "lo" else rank + 1, v[s:s + n].copy())
        ok_halo = bool(np.array_equal(u_loc, u_glob[st.local_to_global]))
        owned = st.owned_global_nodes()
        part = torch.tensor([float((u_glob[owned] ** 2).sum()), float(len(owned))],
                            dtype=torch.float64)
        dist.all_reduce(part)
        results[rank] = (ok_halo, float(part[0]), float(part[1]), float((u_glob ** 2).sum()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["notched16", "lshape"])
def test_halo_protocol_gloo_world2(name):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, results), nprocs=world, join=True)
    n_nodes = MESHES[name]().n_nodes
    for r in range(world):
        ok, s, cnt, ref = results[r]
        assert ok, f"rank {r}: ghost rows differ from the owners' values"
        assert cnt == n_nodes
        assert abs(s - ref) <= 1e-12 * ref


def _gather_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2209_07969_b200 import configs as C
        from paper_2209_07969_b200.schemes import SolverState

        case = C.get_case("tension16")
        mesh = C.build_mesh(case, C.b200_api())
        lay = meshing.StructuredLayout.from_mesh(mesh)
        st = strips.make_strip(lay, world, rank)
        rng = np.random.default_rng(11)
        full = {k: rng.standard_normal(n) for k, n in (
            ("u", 2 * mesh.n_nodes), ("d", mesh.n_nodes), ("d_prev", mesh.n_nodes))}
        gpf = {k: rng.standard_normal((mesh.n_elems, 4)) for k in (
            "tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max")}
        own_nodes = st.owned_global_nodes()
        own_cells = st.cell_local_to_global[st.cell_lo:st.cell_hi]
        own = {"nodes": own_nodes, "cells": own_cells,
               "u": full["u"].reshape(-1, 2)[own_nodes], "d": full["d"][own_nodes],
               "d_prev": full["d_prev"][own_nodes]}
        own.update({k: v[own_cells] for k, v in gpf.items()})

        class _Disc:
            n_u_dofs, n_d_dofs, n_gp = 2 * mesh.n_nodes, mesh.n_nodes, 4

            class mesh_:  # noqa: N801
                n_elems = mesh.n_elems
        _Disc.mesh = _Disc.mesh_
        state = SolverState.zeros(_Disc)
        bench.gather_full(own, state, world)
        ok = (np.array_equal(state.u, full["u"]) and np.array_equal(state.d, full["d"])
              and np.array_equal(state.d_prev, full["d_prev"])
              and all(np.array_equal(getattr(state.gp, k), v) for k, v in gpf.items()))
        results[rank] = ok
    finally:
        dist.destroy_process_group()


def test_bench_gather_full_gloo_world2():
    """bench.py's multi-rank e2e leg rebuilds the full host state from owned strip results."""
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert all(results[r] for r in range(world))
