"""Row-strip domain decomposition of the structured mesh.

Rank r owns the contiguous node rows ``[jlo, jhi)`` (the last rank also owns row ``ny``) and the
cell rows whose lower node row it owns.  Its local mesh is the row-compact sub-mesh of node rows
``[jlo - 1, jhi]`` (one ghost row on each side that exists) plus the slit duplicates when it owns
the slit row.  Because the layout is row-compact, every node row — owned or ghost — is a
contiguous id range both globally and locally, so a halo exchange is two contiguous sends and two
contiguous receives per vector (``ncclSend`` / ``ncclRecv`` over NVLink), and the owned nodes of
a rank are the contiguous local range ``[own_lo, own_hi)`` plus the duplicate block.

Cells of the ghost cell row ``jlo - 1`` are evaluated redundantly from ghost nodal data (same
inputs, same arithmetic -> bit-identical to the owner); Gauss-point history of those cells is kept
consistent the same way, so only nodal rows are ever exchanged.

Cuts are chosen to balance cell counts and never put the first owned row of a rank directly
above the slit row (the rank would then need the duplicates as ghosts).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .meshing import StructuredLayout


@dataclass
class Strip:
    rank: int
    nranks: int
    jlo: int                  # first owned node row (global)
    jhi: int                  # one past the last owned node row (global)
    row0: int                 # first local row (global index) = max(jlo - 1, 0)
    layout: StructuredLayout  # local row-compact layout (rows row0 .. row0 + ny_local)
    local_to_global: np.ndarray
    own_lo: int               # owned local node range [own_lo, own_hi) (+ duplicates)
    own_hi: int
    dup_lo: int               # local id of the first duplicate, = n_local if none
    send_lo: tuple | None     # (local start, count) of owned row jlo, sent to rank - 1
    recv_lo: tuple | None     # (local start, count) of ghost row jlo - 1, from rank - 1
    send_hi: tuple | None     # (local start, count) of owned row jhi - 1, sent to rank + 1
    recv_hi: tuple | None     # (local start, count) of ghost row jhi, from rank + 1
    cell_lo: int              # first OWNED local cell id (the ghost cell row comes first)
    cell_hi: int
    cell_local_to_global: np.ndarray

    @property
    def n_local(self) -> int:
        return self.layout.n_nodes

    def owned_global_nodes(self) -> np.ndarray:
        idx = np.r_[np.arange(self.own_lo, self.own_hi), np.arange(self.dup_lo, self.n_local)]
        return self.local_to_global[idx]


def partition_rows(lay: StructuredLayout, nranks: int, align: int | None = None) -> list:
    """Node-row cuts ``[c_0=0, c_1, ..., c_n=ny+1]`` balancing cell counts.

    Cuts are rounded to a multiple of ``align`` (default: the largest power of two not above a
    quarter of the balanced strip height, at most 512) when that keeps the constraints, so
    every strip's owned sub-mesh coarsens deeply for its local multigrid V-cycle (pf_mgd.cuh);
    a cut never makes the first owned row the slit row or the row directly above it (the rank
    would need the duplicates as ghosts, or its V-cycle would see the lower crack face without
    its cells)."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    ny = lay.ny
    if nranks > (ny + 1) // 2:
        raise ValueError(f"{nranks} strips need at least {2 * nranks} node rows")
    if align is None:
        h = max(1, (ny + 1) // (4 * nranks))
        align = 1
        while align * 2 <= min(h, 512):
            align *= 2
    cells = (lay.elem_hi - lay.elem_lo).astype(np.int64)  # cells of cell row j (owner: row j)
    w = np.r_[cells, 0].astype(float) + 1e-9               # weight of node row j
    cum = np.cumsum(w)
    cuts = [0]

    def ok(c, r):
        hi_lim = ny + 1 - 2 * (nranks - r)
        if c < cuts[-1] + 2 or c > hi_lim:
            return False
        return not (lay.notch_row >= 0 and c in (lay.notch_row, lay.notch_row + 1))

    for r in range(1, nranks):
        c0 = int(np.searchsorted(cum, cum[-1] * r / nranks)) + 1
        cands = []
        if align > 1:
            base = int(round(c0 / align)) * align
            cands += [base, base + align, base - align]
        cands += [c0, c0 + 1, c0 - 1, c0 + 2, c0 - 2]
        hi_lim = ny + 1 - 2 * (nranks - r)
        cands += [min(max(c0, cuts[-1] + 2), hi_lim)]
        c = next((x for x in cands if ok(x, r)), None)
        if c is None:
            raise ValueError(f"cannot cut {ny + 1} node rows into {nranks} strips around the slit")
        cuts.append(c)
    cuts.append(ny + 1)
    if any(b - a < 2 for a, b in zip(cuts, cuts[1:])):
        raise ValueError(f"cannot cut {ny + 1} node rows into {nranks} strips")
    return cuts


def make_strip(lay: StructuredLayout, nranks: int, rank: int, cuts=None) -> Strip:
    cuts = partition_rows(lay, nranks) if cuts is None else cuts
    jlo, jhi = cuts[rank], cuts[rank + 1]
    row0 = max(jlo - 1, 0)
    row1 = min(jhi, lay.ny)  # last local node row (inclusive)
    rows = np.arange(row0, row1 + 1)
    nlo, nhi = lay.node_lo[rows].astype(np.int32), lay.node_hi[rows].astype(np.int32)
    counts = (nhi - nlo).astype(np.int64)
    nstart = np.r_[0, np.cumsum(counts)[:-1]].astype(np.int64)
    n_rows_nodes = int(counts.sum())
    # global ids of the local rows
    l2g = np.concatenate([lay.node_start[j] + np.arange(c) for j, c in zip(rows, counts)]) \
        if n_rows_nodes else np.zeros(0, np.int64)
    # duplicates only when this rank owns the slit row
    has_dup = lay.notch_row >= 0 and jlo <= lay.notch_row < jhi
    notch_row, notch_lo, notch_hi, dup_start = -1, 0, 0, n_rows_nodes
    if has_dup:
        notch_row = lay.notch_row - row0
        notch_lo, notch_hi = lay.notch_lo, lay.notch_hi
        nd = notch_hi - notch_lo
        l2g = np.r_[l2g, lay.dup_start + np.arange(nd)]
    n_local = l2g.size
    # local cell rows: row0 .. row1 - 1
    crow = np.arange(row0, row1)
    elo, ehi = lay.elem_lo[crow].astype(np.int32), lay.elem_hi[crow].astype(np.int32)
    ecount = (ehi - elo).astype(np.int64)
    estart = np.r_[0, np.cumsum(ecount)[:-1]].astype(np.int64)
    cl2g = np.concatenate([lay.elem_start[j] + np.arange(c) for j, c in zip(crow, ecount)]) \
        if ecount.sum() else np.zeros(0, np.int64)
    local = StructuredLayout(
        nx=lay.nx, ny=int(row1 - row0), hx=lay.hx, hy=lay.hy,
        node_lo=nlo, node_hi=nhi, node_start=nstart,
        elem_lo=elo, elem_hi=ehi, elem_start=estart,
        notch_row=notch_row, notch_lo=notch_lo, notch_hi=notch_hi,
        dup_start=dup_start if has_dup else 0, n_nodes=int(n_local),
        n_elems=int(ecount.sum()))
    row_range = lambda j: (int(nstart[j - row0]), int(counts[j - row0]))  # noqa: E731
    own_lo = row_range(jlo)[0]
    last = jhi - 1
    own_hi = row_range(last)[0] + row_range(last)[1]
    ghost_cells = int(ecount[0]) if jlo > 0 else 0
    return Strip(
        rank=rank, nranks=nranks, jlo=jlo, jhi=jhi, row0=row0, layout=local,
        local_to_global=l2g, own_lo=own_lo, own_hi=own_hi,
        dup_lo=dup_start if has_dup else n_local,
        send_lo=row_range(jlo) if rank > 0 else None,
        recv_lo=row_range(jlo - 1) if rank > 0 else None,
        send_hi=row_range(jhi - 1) if rank < nranks - 1 else None,
        recv_hi=row_range(jhi) if rank < nranks - 1 else None,
        cell_lo=ghost_cells, cell_hi=int(ecount.sum()), cell_local_to_global=cl2g)


def halo_exchange(strip: Strip, vec: np.ndarray, comps: int, send, recv) -> None:
    """Reference implementation of one halo exchange on host arrays (tests and documentation
    of the device protocol): ``send(dst_rank, array)`` / ``recv(src_rank, n) -> array``.
    Order: exchange with the lower neighbour first, then the upper one (both directions)."""
    v = vec.reshape(-1, comps)
    if strip.send_lo is not None:
        s, n = strip.send_lo
        send(strip.rank - 1, v[s:s + n].copy())
    if strip.send_hi is not None:
        s, n = strip.send_hi
        send(strip.rank + 1, v[s:s + n].copy())
    if strip.recv_lo is not None:
        s, n = strip.recv_lo
        v[s:s + n] = recv(strip.rank - 1, n * comps).reshape(n, comps)
    if strip.recv_hi is not None:
        s, n = strip.recv_hi
        v[s:s + n] = recv(strip.rank + 1, n * comps).reshape(n, comps)
