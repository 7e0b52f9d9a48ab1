"""Structured Q4 meshes and their row-compact device layout.

The builders reproduce, array for array, the reference's ``build_notched_square``
(``meshing.py:90-151``) and ``build_lshape_mesh`` (``meshing.py:159-215``) — same node order
(row-major ``j*(nx+1)+i``, slit duplicates appended), same CCW connectivity, same boundary
tags — but vectorised, so the 8192^2 multi-crack mesh (config 5) builds in seconds instead of
a 67 M-iteration Python loop.

``StructuredLayout.from_mesh`` recovers the row-compact description the kernels use
(``include/pf_b200.h``: ``pf_mesh``) from ANY mesh object with ``nodes`` / ``elements``
arrays (ours or the reference's) and verifies every element's connectivity against it, so a
mesh the device path cannot represent exactly is rejected with ``ValueError`` instead of
being solved wrongly.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Mesh:
    nodes: np.ndarray
    elements: np.ndarray
    boundary_sets: dict = field(default_factory=dict)
    notch: dict | None = None

    @property
    def n_nodes(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def n_elems(self) -> int:
        return int(self.elements.shape[0])

    @property
    def dim(self) -> int:
        return int(self.nodes.shape[1])

    def validate(self) -> None:
        if not np.all(np.isfinite(self.nodes)):
            raise ValueError("non-finite node coordinates")
        if self.elements.min() < 0 or self.elements.max() >= self.n_nodes:
            raise ValueError("element references a missing node")
        for tag, idx in self.boundary_sets.items():
            if len(idx) and (idx.min() < 0 or idx.max() >= self.n_nodes):
                raise ValueError(f"boundary set {tag!r} references a missing node")


def select_boundary(mesh: Mesh, tag: str) -> np.ndarray:
    try:
        return mesh.boundary_sets[tag]
    except KeyError:
        known = ", ".join(sorted(mesh.boundary_sets))
        raise KeyError(f"unknown boundary tag {tag!r}; known tags: {known}") from None


def _grid_cells(nx: int, ny: int, ids: np.ndarray) -> np.ndarray:
    """CCW connectivity of an nx x ny cell grid given the (ny+1, nx+1) node-id table."""
    return np.stack([ids[:-1, :-1], ids[:-1, 1:], ids[1:, 1:], ids[1:, :-1]], axis=-1)


def build_notched_square(nx: int, ny: int, side: float,
                         notch_from_left_to_center: bool = True) -> Mesh:
    if nx < 2 or ny < 2 or nx % 2 or ny % 2:
        raise ValueError("nx and ny must be even and >= 2 so the notch lies on edges")
    if side <= 0.0:
        raise ValueError("side must be positive")
    xs = np.linspace(0.0, side, nx + 1)
    ys = np.linspace(0.0, side, ny + 1)
    xg, yg = np.meshgrid(xs, ys, indexing="xy")
    nodes = np.column_stack([xg.ravel(), yg.ravel()])
    ids = np.arange((nx + 1) * (ny + 1), dtype=np.int64).reshape(ny + 1, nx + 1)
    elems = _grid_cells(nx, ny, ids).reshape(-1, 4)
    notch = None
    if notch_from_left_to_center:
        mj, mi = ny // 2, nx // 2
        base = ids[mj, :mi]
        dup = nodes.shape[0] + np.arange(mi, dtype=np.int64)
        nodes = np.vstack([nodes, nodes[base]])
        row = elems[mj * nx: mj * nx + mi]  # cells just above the slit, columns < tip
        lut = np.full(ids.size, -1, dtype=np.int64)
        lut[base] = dup
        remap = lut[row]
        elems[mj * nx: mj * nx + mi] = np.where(remap >= 0, remap, row)
        notch = {"line": ((0.0, side / 2.0), (side / 2.0, side / 2.0)),
                 "pairs": list(zip(base.tolist(), dup.tolist()))}
    tol = 1e-12 * max(side, 1.0)
    bsets = {
        "bottom": np.flatnonzero(np.abs(nodes[:, 1]) < tol),
        "top": np.flatnonzero(np.abs(nodes[:, 1] - side) < tol),
        "left": np.flatnonzero(np.abs(nodes[:, 0]) < tol),
        "right": np.flatnonzero(np.abs(nodes[:, 0] - side) < tol),
    }
    return Mesh(nodes=nodes, elements=elems, boundary_sets=bsets, notch=notch)


L_PANEL_SIZE = 500.0
L_PANEL_CUTOUT = 250.0
L_LOAD_STRIP = 30.0


def build_lshape_mesh(h: float) -> Mesh:
    arm = L_PANEL_SIZE - L_PANEL_CUTOUT
    n_arm = arm / h
    if abs(n_arm - round(n_arm)) > 1e-9 or round(n_arm) < 1:
        raise ValueError(f"element size {h} does not divide the arm dimension {arm}")
    n = int(round(L_PANEL_SIZE / h))
    xs = np.linspace(0.0, L_PANEL_SIZE, n + 1)
    centre = 0.5 * (xs[:-1] + xs[1:])
    keep_cell = ~((centre[None, :] > L_PANEL_CUTOUT) & (centre[:, None] < L_PANEL_CUTOUT))
    cj, ci = np.nonzero(keep_cell)  # row-major (j outer, i inner) like the reference loop
    gid = np.arange((n + 1) * (n + 1), dtype=np.int64).reshape(n + 1, n + 1)
    corners = np.stack([gid[cj, ci], gid[cj, ci + 1], gid[cj + 1, ci + 1], gid[cj + 1, ci]], -1)
    keep_node = np.zeros(gid.size, dtype=bool)
    keep_node[corners.ravel()] = True
    kept = np.flatnonzero(keep_node)
    renum = np.full(gid.size, -1, dtype=np.int64)
    renum[kept] = np.arange(kept.size)
    coords = np.column_stack([xs[kept % (n + 1)], xs[kept // (n + 1)]])
    elems = renum[corners]
    tol = 1e-9 * L_PANEL_SIZE
    bottom = np.flatnonzero(np.abs(coords[:, 1]) < tol)
    on_arm = (np.abs(coords[:, 1] - L_PANEL_CUTOUT) < tol) & (coords[:, 0] > L_PANEL_CUTOUT + tol)
    near_tip = coords[:, 0] >= L_PANEL_SIZE - max(L_LOAD_STRIP, h) - tol
    return Mesh(nodes=coords, elements=elems,
                boundary_sets={"bottom_clamp": bottom, "load_zone": np.flatnonzero(on_arm & near_tip)})


# -------------------------------------------------------------------------------------------
@dataclass
class StructuredLayout:
    """Row-compact structured description of a uniform-rectangle Q4 mesh (``pf_mesh``)."""

    nx: int
    ny: int
    hx: float
    hy: float
    node_lo: np.ndarray
    node_hi: np.ndarray
    node_start: np.ndarray
    elem_lo: np.ndarray
    elem_hi: np.ndarray
    elem_start: np.ndarray
    notch_row: int
    notch_lo: int
    notch_hi: int
    dup_start: int
    n_nodes: int
    n_elems: int

    @classmethod
    def from_mesh(cls, mesh) -> "StructuredLayout":
        nodes = np.asarray(mesh.nodes, dtype=np.float64)
        elems = np.asarray(mesh.elements, dtype=np.int64)
        if nodes.ndim != 2 or nodes.shape[1] != 2 or elems.ndim != 2 or elems.shape[1] != 4:
            raise ValueError("only 2-D 4-node quadrilateral meshes are supported")
        nn, ne = nodes.shape[0], elems.shape[0]
        if ne == 0:
            raise ValueError("empty mesh")
        x0, y0 = nodes[:, 0].min(), nodes[:, 1].min()
        c = nodes[elems]  # (ne, 4, 2)
        hx = float(c[0, 1, 0] - c[0, 0, 0])
        hy = float(c[0, 3, 1] - c[0, 0, 1])
        if not (hx > 0.0 and hy > 0.0):
            raise ValueError("non-positive jacobian in element 0")
        scale = max(float(np.abs(nodes).max()), hx, hy)
        tol = 1e-9 * scale
        # every element must be an axis-aligned CCW rectangle hx x hy
        ex = np.array([0.0, hx, hx, 0.0])
        ey = np.array([0.0, 0.0, hy, hy])
        if (np.abs(c[:, :, 0] - c[:, :1, 0] - ex).max() > tol or
                np.abs(c[:, :, 1] - c[:, :1, 1] - ey).max() > tol):
            raise ValueError("the B200 path needs uniform axis-aligned rectangular cells "
                             "(SURVEY.md App. C.1)")
        gi = np.rint((nodes[:, 0] - x0) / hx).astype(np.int64)
        gj = np.rint((nodes[:, 1] - y0) / hy).astype(np.int64)
        if (np.abs(x0 + gi * hx - nodes[:, 0]).max() > tol or
                np.abs(y0 + gj * hy - nodes[:, 1]).max() > tol):
            raise ValueError("nodes are not on a uniform grid")
        nx, ny = int(gi.max()), int(gj.max())
        # regular nodes come first, row-major and compact; duplicates (slit) trail
        key = gj * (nx + 1) + gi
        # a node is a duplicate iff an earlier node has the same grid position
        _, first_idx = np.unique(key, return_index=True)
        is_dup = np.ones(nn, dtype=bool)
        is_dup[first_idx] = False
        n_reg = int((~is_dup).sum())
        if is_dup[:n_reg].any() or (~is_dup[n_reg:]).any():
            raise ValueError("duplicate nodes must trail the regular nodes")
        rk = key[:n_reg]
        if n_reg > 1 and np.any(np.diff(rk) <= 0):
            raise ValueError("regular nodes are not numbered row-major")
        rj, ri = gj[:n_reg], gi[:n_reg]
        node_lo = np.zeros(ny + 1, np.int32)
        node_hi = np.zeros(ny + 1, np.int32)
        node_start = np.zeros(ny + 1, np.int64)
        counts = np.bincount(rj, minlength=ny + 1)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
        for j in np.flatnonzero(counts):
            s, n_j = int(starts[j]), int(counts[j])
            lo, hi = int(ri[s]), int(ri[s + n_j - 1]) + 1
            if hi - lo != n_j:
                raise ValueError(f"node row {j} is not contiguous")
            node_lo[j], node_hi[j], node_start[j] = lo, hi, s
        notch_row, notch_lo, notch_hi, dup_start = -1, 0, 0, 0
        if n_reg < nn:
            dj, di = gj[n_reg:], gi[n_reg:]
            if np.any(dj != dj[0]) or np.any(np.diff(di) != 1):
                raise ValueError("duplicate nodes must form one contiguous slit row")
            notch_row, notch_lo, notch_hi, dup_start = int(dj[0]), int(di[0]), int(di[-1]) + 1, n_reg
        # cells: row-major compact by their lower-left corner
        ci = np.rint((c[:, 0, 0] - x0) / hx).astype(np.int64)
        cj = np.rint((c[:, 0, 1] - y0) / hy).astype(np.int64)
        ck = cj * nx + ci
        if ne > 1 and np.any(np.diff(ck) <= 0):
            raise ValueError("cells are not numbered row-major")
        elem_lo = np.zeros(ny, np.int32)
        elem_hi = np.zeros(ny, np.int32)
        elem_start = np.zeros(ny, np.int64)
        ecounts = np.bincount(cj, minlength=ny)
        estarts = np.concatenate([[0], np.cumsum(ecounts)[:-1]])
        for j in np.flatnonzero(ecounts):
            s, n_j = int(estarts[j]), int(ecounts[j])
            lo, hi = int(ci[s]), int(ci[s + n_j - 1]) + 1
            if hi - lo != n_j:
                raise ValueError(f"cell row {j} is not contiguous")
            elem_lo[j], elem_hi[j], elem_start[j] = lo, hi, s
        lay = cls(nx, ny, hx, hy, node_lo, node_hi, node_start, elem_lo, elem_hi, elem_start,
                  notch_row, notch_lo, notch_hi, dup_start, nn, ne)
        if not np.array_equal(lay.connectivity(), elems):
            raise ValueError("element connectivity does not match the structured layout")
        return lay

    @classmethod
    def rectangle(cls, nx: int, ny: int, hx: float, hy: float) -> "StructuredLayout":
        """Layout of a plain nx x ny grid (build_notched_square(..., notch=False)) built
        directly, without materialising node / element arrays (config 5: 67 M cells)."""
        rows = np.arange(ny + 1, dtype=np.int64)
        return cls(nx, ny, hx, hy,
                   np.zeros(ny + 1, np.int32), np.full(ny + 1, nx + 1, np.int32),
                   rows * (nx + 1), np.zeros(ny, np.int32), np.full(ny, nx, np.int32),
                   rows[:ny] * nx, -1, 0, 0, 0, (nx + 1) * (ny + 1), nx * ny)

    def node_id(self, i, j):
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        return self.node_start[j] + (i - self.node_lo[j])

    def connectivity(self) -> np.ndarray:
        """Element -> node ids implied by the layout (the kernels' arithmetic, vectorised)."""
        rows = np.repeat(np.arange(self.ny), self.elem_hi - self.elem_lo)
        cols = np.concatenate([np.arange(lo, hi) for lo, hi in zip(self.elem_lo, self.elem_hi)]) \
            if self.n_elems else np.zeros(0, np.int64)
        n0 = self.node_id(cols, rows)
        n1 = self.node_id(cols + 1, rows)
        n2 = self.node_id(cols + 1, rows + 1)
        n3 = self.node_id(cols, rows + 1)
        if self.notch_row >= 0:
            sel = rows == self.notch_row
            for nid, col in ((n0, cols), (n1, cols + 1)):
                m = sel & (col >= self.notch_lo) & (col < self.notch_hi)
                nid[m] = self.dup_start + (col[m] - self.notch_lo)
        return np.stack([n0, n1, n2, n3], axis=1)
