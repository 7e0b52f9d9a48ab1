"""Row-strip multi-GPU sessions: one process (or host thread) per strip.

``StripSession`` wraps a ``DeviceSession`` created on the strip's LOCAL sub-mesh
(``strips.make_strip``) with ``pf_create_strip``; it maps global state, boundary conditions,
pins and reaction node sets to local ids, and gathers owned results back.  Communication:

* ``comm="nccl"``: NCCL over NVLink / NVSwitch, one process per GPU (``torchrun``); rank 0's
  ``ncclUniqueId`` is broadcast with ``torch.distributed`` (``nccl_unique_id`` +
  ``broadcast_object_list``).
* ``comm=HostGroup``: in-process emulation of several strips on ONE GPU, one host thread per
  strip (tests).  Kernels never wait on each other; the threads meet on the host.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from .meshing import StructuredLayout
from .session import DeviceSession, pack_bcs  # noqa: F401
from .strips import Strip, make_strip, partition_rows


def nccl_lib_path() -> str | None:
    try:
        import nvidia.nccl  # noqa: PLC0415

        base = list(nvidia.nccl.__path__)[0]
        cand = os.path.join(base, "lib", "libnccl.so.2")
        return cand if os.path.exists(cand) else None
    except Exception:  # noqa: BLE001
        return None


def nccl_unique_id() -> bytes:
    lib = N.load()
    if "PFB200_NCCL_LIB" not in os.environ and nccl_lib_path():
        os.environ["PFB200_NCCL_LIB"] = nccl_lib_path()
    buf = (C.c_ubyte * 128)()
    st = lib.pf_nccl_unique_id(C.byref(buf))
    if st != N.PF_OK:
        raise RuntimeError("pf_nccl_unique_id failed (NCCL not loadable)")
    return bytes(buf)


class HostGroup:
    """In-process communicator for ``nranks`` strips driven by ``nranks`` host threads."""

    def __init__(self, nranks: int):
        self.lib = N.load()
        self.nranks = nranks
        h = C.c_void_p()
        if self.lib.pf_host_group_create(nranks, C.byref(h)) != N.PF_OK:
            raise RuntimeError("pf_host_group_create failed")
        self.h = h

    def close(self):
        if self.h is not None:
            self.lib.pf_host_group_destroy(self.h)
            self.h = None


class StripSession:
    def __init__(self, mesh_or_layout, params, config, rank: int, nranks: int, comm,
                 device: int = 0, nccl_id: bytes | None = None, cuts=None):
        lay = (mesh_or_layout if isinstance(mesh_or_layout, StructuredLayout)
               else StructuredLayout.from_mesh(mesh_or_layout))
        self.glob = lay
        cuts = partition_rows(lay, nranks) if cuts is None else cuts
        self.strip: Strip = make_strip(lay, nranks, rank, cuts)
        st = self.strip
        ps = N.PfStrip()
        ps.rank, ps.nranks = rank, nranks
        ps.own_lo, ps.own_hi, ps.dup_lo = st.own_lo, st.own_hi, st.dup_lo
        ps.cell_lo, ps.cell_hi = st.cell_lo, st.cell_hi
        for side in ("lo", "hi"):
            for kind in ("send", "recv"):
                rng = getattr(st, f"{kind}_{side}")
                start, count = rng if rng is not None else (0, 0)
                setattr(ps, f"{kind}_{side}_start", start)
                setattr(ps, f"{kind}_{side}_count", count)
        if comm == "nccl":
            if "PFB200_NCCL_LIB" not in os.environ and nccl_lib_path():
                os.environ["PFB200_NCCL_LIB"] = nccl_lib_path()
            if nccl_id is None:
                raise ValueError("comm='nccl' needs the broadcast ncclUniqueId")
            ps.comm_kind = 0
            C.memmove(ps.nccl_id, nccl_id, 128)
        else:
            ps.comm_kind = 1
            ps.host_group = comm.h
        self.sess = DeviceSession(st.layout, params, config, device=device, strip=ps)
        # global -> local id maps (all local nodes incl. ghosts / owned only)
        self.l2g = st.local_to_global
        self.g2l = np.full(lay.n_nodes, -1, dtype=np.int64)
        self.g2l[self.l2g] = np.arange(self.l2g.size)
        owned = np.zeros(self.l2g.size, bool)
        owned[st.own_lo:st.own_hi] = True
        owned[st.dup_lo:] = True
        self.owned_local = owned
        self.cl2g = st.cell_local_to_global

    # -- maps ------------------------------------------------------------------------------
    def local_dofs(self, dofs):
        dofs = np.asarray(dofs, dtype=np.int64)
        loc = self.g2l[dofs // 2]
        keep = loc >= 0
        return 2 * loc[keep] + dofs[keep] % 2

    def local_bcs(self, bc_increments):
        return [(self.local_dofs(d), inc) for d, inc in bc_increments]

    def local_nodes(self, nodes, owned_only=False):
        loc = self.g2l[np.asarray(nodes, dtype=np.int64)]
        loc = loc[loc >= 0]
        return loc[self.owned_local[loc]] if owned_only else loc

    # -- state -----------------------------------------------------------------------------
    def push_global(self, u, d, d_prev, trp, dev2, psi, psimax):
        n, c = self.l2g, self.cl2g
        self.sess.push(np.asarray(u).reshape(-1, 2)[n].ravel(), np.asarray(d)[n],
                       np.asarray(d_prev)[n], *(np.asarray(a).reshape(-1, 4)[c]
                                                for a in (trp, dev2, psi, psimax)))

    def owned_state(self) -> dict:
        """Owned nodal / cell results with their global ids."""
        loc = self.sess.pull()
        own = np.flatnonzero(self.owned_local)
        st = self.strip
        cells = np.arange(st.cell_lo, st.cell_hi)
        out = {"nodes": self.l2g[own], "cells": self.cl2g[cells],
               "u": loc["u"].reshape(-1, 2)[own], "d": loc["d"][own],
               "d_prev": loc["d_prev"][own]}
        for k in ("tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max"):
            out[k] = loc[k][cells]
        return out

    # -- hot path --------------------------------------------------------------------------
    def step(self, scheme, bc_increments, pinned_d_nodes=None):
        pins = None if pinned_d_nodes is None else self.local_nodes(pinned_d_nodes)
        return self.sess.step(scheme, self.local_bcs(bc_increments), pins)

    def reaction_force(self, node_set, component: int) -> float:
        return self.sess.reaction_force(self.local_nodes(node_set, owned_only=True), component)

    def close(self):
        self.sess.close()
