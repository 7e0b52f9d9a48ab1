"""Load cases (BASELINE configs 1-5 and their reduced analogues) and a load-step runner.

The reference ships no runner and no boundary-condition builders (SURVEY.md §8(c) "Missing
pieces", Appendix B).  This module is the single definition of those recipes; it is used,
unchanged, by

* ``tests/golden/make_golden.py`` to drive the *unmodified* reference package
  (``/root/reference/pkg/src/phasefrac``) and record golden tables,
* the CPU oracle (``oracle/``) in the parity tests, and
* the B200 path (``paper_2209_07969_b200``) in the tests and in ``bench.py``.

Every recipe is expressed against an *API namespace* exposing the reference's public names
(``build_notched_square``, ``build_lshape_mesh``, ``MaterialParams``, ``SolverConfig``,
``SchemeKind``, ``Discretization``, ``SolverState``, ``staggered_step``, ``reaction_force``),
so the same code drives the reference, the oracle and the GPU drop-in.

Reference anchors:
  * per-step call ``staggered_step(disc, state, scheme, bc, params, cfg, pins)``
    (``schemes.py:332-340``), reaction via ``reaction_force`` (``assembly.py:315-326``);
  * DOF numbering ``2*node + comp`` (``assembly.py:272-276``);
  * boundary tags of ``build_notched_square`` (``meshing.py:141-147``) and
    ``build_lshape_mesh`` (``meshing.py:207-214``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace
from types import SimpleNamespace

import numpy as np


@dataclass(frozen=True)
class LoadCase:
    """One benchmark configuration."""

    name: str
    mesh: tuple  # ("notched", nx, ny, side, notch) | ("lshape", h)
    material: dict  # kwargs of MaterialParams.from_young_poisson
    loading: str  # "tension" | "shear" | "lpanel" | "biaxial"
    inc: float  # displacement increment per load step (mm)
    n_steps: int
    schemes: tuple = ("ST", "S1")
    tol_st: float = 1.0e-5
    # (n_cracks, seed, len_lo, len_hi) for seeded straight pre-cracks (config 5)
    precracks: tuple | None = None
    note: str = ""

    @property
    def dofs_note(self) -> str:
        return self.note


_TENSION_MAT = dict(e_mod=210000.0, nu=0.3, g_c=2.7, length_l=0.015, at_model="AT2")

CASES: dict[str, LoadCase] = {}


def _add(case: LoadCase) -> LoadCase:
    CASES[case.name] = case
    return case


# --- BASELINE.json configs -----------------------------------------
_add(LoadCase("cfg1", ("notched", 64, 64, 1.0, True), _TENSION_MAT, "tension", 1.0e-4, 65,
              ("ST", "S1", "S2", "S3"), note="BASELINE configs[0]: 64x64 tension, CPU-runnable"))
_add(LoadCase("cfg2", ("notched", 512, 512, 1.0, True), {**_TENSION_MAT, "length_l": 0.0075},
              "tension", 1.0e-4, 65, ("ST", "S1", "S2", "S3"),
              note="BASELINE configs[1]: 512x512 tension, l=0.0075"))
_add(LoadCase("cfg3", ("notched", 1024, 1024, 1.0, True), {**_TENSION_MAT, "length_l": 0.0075},
              "shear", 1.0e-4, 150, ("ST", "S1", "S2", "S3"),
              note="BASELINE configs[2]: 1024x1024 shear"))
_add(LoadCase("cfg4", ("lshape", 0.5),
              dict(e_mod=25850.0, nu=0.18, g_c=0.089, length_l=2.0, at_model="AT2"),
              "lpanel", 2.0e-3, 500, ("ST", "S1"), note="BASELINE configs[3]: L-panel h=0.5"))
_add(LoadCase("cfg5", ("notched", 8192, 8192, 1000.0, False),
              dict(e_mod=10000.0, nu=0.25, g_c=0.01, length_l=2.0, at_model="AT2"),
              "biaxial", 2.0e-3, 50, ("ST", "S1"), precracks=(256, 20220916, 5.0, 20.0),
              note="BASELINE configs[4]: 8192^2 multi-crack biaxial"))

# --- reduced analogues (identical runner logic, sizes the CPU reference finishes) ---------
_add(LoadCase("tension16", ("notched", 16, 16, 1.0, True), {**_TENSION_MAT, "length_l": 0.08},
              "tension", 6.0e-4, 16, ("ST", "S1", "S2", "S3"),
              note="cfg1/cfg2 analogue, cracks within 16 steps"))
_add(LoadCase("tension16_at1", ("notched", 16, 16, 1.0, True),
              {**_TENSION_MAT, "length_l": 0.08, "at_model": "AT1"},
              "tension", 6.0e-4, 16, ("ST", "S1", "S3"),
              note="AT1 (the reference default model) on the tension16 analogue"))
_add(LoadCase("tension32", ("notched", 32, 32, 1.0, True), {**_TENSION_MAT, "length_l": 0.04},
              "tension", 4.0e-4, 18, ("ST", "S1", "S2", "S3"), note="cfg2 analogue"))
_add(LoadCase("shear32", ("notched", 32, 32, 1.0, True), {**_TENSION_MAT, "length_l": 0.04},
              "shear", 5.0e-4, 22, ("ST", "S1", "S2", "S3"), note="cfg3 analogue"))
_add(LoadCase("lpanel25", ("lshape", 25.0),
              dict(e_mod=25850.0, nu=0.18, g_c=0.089, length_l=40.0, at_model="AT2"),
              "lpanel", 0.1, 12, ("ST", "S1"), note="cfg4 analogue (20x20 bounding grid)"))
_add(LoadCase("multicrack256", ("notched", 256, 256, 1000.0, False),
              dict(e_mod=10000.0, nu=0.25, g_c=0.01, length_l=2.0, at_model="AT2"),
              "biaxial", 2.0e-3, 50, ("ST", "S1"), precracks=(8, 20220916, 5.0, 20.0),
              note="cfg5 analogue of SURVEY.md App. B (256^2, 8 cracks, same seed logic)"))
_add(LoadCase("multicrack32", ("notched", 32, 32, 1000.0, False),
              dict(e_mod=10000.0, nu=0.25, g_c=0.01, length_l=60.0, at_model="AT2"),
              "biaxial", 0.1, 10, ("ST", "S1"), precracks=(6, 20220916, 60.0, 160.0),
              note="cfg5 analogue"))


def get_case(name: str, **overrides) -> LoadCase:
    case = CASES[name]
    return replace(case, **overrides) if overrides else case


# -------------------------------------------------------------------------------------------
# API namespaces
# -------------------------------------------------------------------------------------------
def reference_api(src: str = "/root/reference/pkg/src") -> SimpleNamespace:
    """The unmodified reference package as an API namespace (only in the build container)."""
    import sys

    if src not in sys.path:
        sys.path.insert(0, src)
    from phasefrac import assembly, material, meshing, schemes  # noqa: PLC0415

    return SimpleNamespace(
        name="reference",
        build_notched_square=meshing.build_notched_square,
        build_lshape_mesh=meshing.build_lshape_mesh,
        MaterialParams=material.MaterialParams,
        SolverConfig=schemes.SolverConfig,
        SchemeKind=schemes.SchemeKind,
        Discretization=assembly.Discretization,
        SolverState=schemes.SolverState,
        staggered_step=schemes.staggered_step,
        reaction_force=assembly.reaction_force,
    )


def b200_api() -> SimpleNamespace:
    """The B200 drop-in as an API namespace."""
    from . import assembly, material, meshing, schemes  # noqa: PLC0415

    return SimpleNamespace(
        name="b200",
        build_notched_square=meshing.build_notched_square,
        build_lshape_mesh=meshing.build_lshape_mesh,
        MaterialParams=material.MaterialParams,
        SolverConfig=schemes.SolverConfig,
        SchemeKind=schemes.SchemeKind,
        Discretization=assembly.Discretization,
        SolverState=schemes.SolverState,
        staggered_step=schemes.staggered_step,
        reaction_force=assembly.reaction_force,
    )


# -------------------------------------------------------------------------------------------
# recipes
# -------------------------------------------------------------------------------------------
def build_mesh(case: LoadCase, api):
    kind = case.mesh[0]
    if kind == "notched":
        _, nx, ny, side, notch = case.mesh
        return api.build_notched_square(nx, ny, side, notch_from_left_to_center=notch)
    if kind == "lshape":
        return api.build_lshape_mesh(case.mesh[1])
    raise ValueError(f"unknown mesh kind {kind!r}")


def material(case: LoadCase, api):
    m = dict(case.material)
    return api.MaterialParams.from_young_poisson(m.pop("e_mod"), m.pop("nu"), **m)


def _dofs(nodes, comp):
    return 2 * np.asarray(nodes, dtype=np.int64) + comp


def boundary_conditions(case: LoadCase, mesh) -> list:
    """``[(dof_array, increment), ...]`` for one load step."""
    b = mesh.boundary_sets
    if case.loading == "tension":  # bottom fixed; top ux = 0, uy += inc
        return [(_dofs(b["bottom"], 0), 0.0), (_dofs(b["bottom"], 1), 0.0),
                (_dofs(b["top"], 0), 0.0), (_dofs(b["top"], 1), case.inc)]
    if case.loading == "shear":  # bottom fixed; left/right uy = 0; top uy = 0, ux += inc
        return [(_dofs(b["bottom"], 0), 0.0), (_dofs(b["bottom"], 1), 0.0),
                (_dofs(b["left"], 1), 0.0), (_dofs(b["right"], 1), 0.0),
                (_dofs(b["top"], 1), 0.0), (_dofs(b["top"], 0), case.inc)]
    if case.loading == "lpanel":  # bottom clamp; load zone uy += inc
        return [(_dofs(b["bottom_clamp"], 0), 0.0), (_dofs(b["bottom_clamp"], 1), 0.0),
                (_dofs(b["load_zone"], 1), case.inc)]
    if case.loading == "biaxial":  # left ux = 0, bottom uy = 0, right ux += inc, top uy += inc
        return [(_dofs(b["left"], 0), 0.0), (_dofs(b["bottom"], 1), 0.0),
                (_dofs(b["right"], 0), case.inc), (_dofs(b["top"], 1), case.inc)]
    raise ValueError(f"unknown loading {case.loading!r}")


def pinned_nodes(case: LoadCase, mesh):
    if case.loading == "lpanel":
        return np.asarray(mesh.boundary_sets["load_zone"], dtype=np.int64)
    return None


def reaction_sets(case: LoadCase, mesh) -> list:
    """``[(label, node_set, component), ...]`` reported per step."""
    b = mesh.boundary_sets
    if case.loading == "tension":
        return [("top_y", b["top"], 1)]
    if case.loading == "shear":
        return [("top_x", b["top"], 0)]
    if case.loading == "lpanel":
        return [("load_y", b["load_zone"], 1)]
    if case.loading == "biaxial":
        return [("right_x", b["right"], 0), ("top_y", b["top"], 1)]
    raise ValueError(case.loading)


def precrack_segments(case: LoadCase) -> tuple:
    """The seeded straight pre-cracks as end points [(ax, ay, bx, by), ...]
    and the marking radius h/2.

    Draw order from ``np.random.default_rng(seed)``: centres U[0, side]^2, then lengths
    U[len_lo, len_hi], then angles U[0, pi).
    """
    if case.precracks is None:
        return np.zeros((0, 4)), 0.0
    n, seed, lo, hi = case.precracks
    _, nx, ny, side, _ = case.mesh
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, side, size=(n, 2))
    lengths = rng.uniform(lo, hi, size=n)
    angles = rng.uniform(0.0, np.pi, size=n)
    segs = []
    for (cx, cy), ln, th in zip(centres, lengths, angles):
        dx, dy = 0.5 * ln * np.cos(th), 0.5 * ln * np.sin(th)
        segs.append((cx - dx, cy - dy, cx + dx, cy + dy))
    return np.array(segs, dtype=np.float64).reshape(-1, 4), 0.5 * (side / nx)


def precrack_nodes(case: LoadCase, mesh) -> np.ndarray:
    """Nodes within h/2 of one of the seeded straight pre-cracks (precrack_segments); the
    host reference of the device initialiser (DeviceSession.init_state / pf_init_state)."""
    if case.precracks is None:
        return np.zeros(0, dtype=np.int64)
    _, nx, ny, side, _ = case.mesh
    segs, _ = precrack_segments(case)
    h = side / nx
    coords = np.asarray(mesh.nodes)
    # regular-grid lookup (column i, row j) -> node ids; a slit position of a notched square
    # holds two nodes (the crack faces share the coordinates) and both are tested
    gi = np.rint(coords[:, 0] / h).astype(np.int64)
    gj = np.rint(coords[:, 1] / h).astype(np.int64)
    key = gj * (nx + 1) + gi
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.r_[True, ks[1:] != ks[:-1]]
    lut = np.full((2, (ny + 1) * (nx + 1)), -1, dtype=np.int64)
    lut[0, ks[first]] = order[first]
    lut[1, ks[~first]] = order[~first]
    lut = lut.reshape(2, ny + 1, nx + 1)
    hit = np.zeros(coords.shape[0], dtype=bool)
    for ax, ay, bx, by in segs:
        i0 = max(int(np.floor((min(ax, bx) - h) / h)), 0)
        i1 = min(int(np.ceil((max(ax, bx) + h) / h)), nx)
        j0 = max(int(np.floor((min(ay, by) - h) / h)), 0)
        j1 = min(int(np.ceil((max(ay, by) + h) / h)), ny)
        ids = lut[:, j0:j1 + 1, i0:i1 + 1].ravel()
        ids = ids[ids >= 0]
        px, py = coords[ids, 0], coords[ids, 1]
        ex, ey = bx - ax, by - ay
        t = np.clip(((px - ax) * ex + (py - ay) * ey) / (ex * ex + ey * ey), 0.0, 1.0)
        dist = np.hypot(px - (ax + t * ex), py - (ay + t * ey))
        hit[ids[dist <= 0.5 * h]] = True
    return np.flatnonzero(hit)


def precrack_nodes_grid(case: LoadCase) -> np.ndarray:
    """precrack_nodes for the plain square of a case (build_notched_square(..., notch=False))
    from its grid coordinates (np.linspace, like the mesh builder) without materialising the node
    array (config 5: 67 M nodes); node (i, j) has id j (nx + 1) + i."""
    if case.precracks is None:
        return np.zeros(0, dtype=np.int64)
    _, nx, ny, side, notch = case.mesh
    if notch:
        raise ValueError("precrack_nodes_grid: plain squares only")
    xs = np.linspace(0.0, side, nx + 1)
    ys = np.linspace(0.0, side, ny + 1)
    segs, _ = precrack_segments(case)
    h = side / nx
    hit = []
    for ax, ay, bx, by in segs:
        i0 = max(int(np.floor((min(ax, bx) - h) / h)), 0)
        i1 = min(int(np.ceil((max(ax, bx) + h) / h)), nx)
        j0 = max(int(np.floor((min(ay, by) - h) / h)), 0)
        j1 = min(int(np.ceil((max(ay, by) + h) / h)), ny)
        jj, ii = np.meshgrid(np.arange(j0, j1 + 1), np.arange(i0, i1 + 1), indexing="ij")
        px, py = xs[ii.ravel()], ys[jj.ravel()]
        ex, ey = bx - ax, by - ay
        t = np.clip(((px - ax) * ex + (py - ay) * ey) / (ex * ex + ey * ey), 0.0, 1.0)
        dist = np.hypot(px - (ax + t * ex), py - (ay + t * ey))
        ids = jj.ravel() * (nx + 1) + ii.ravel()
        hit.append(ids[dist <= 0.5 * h])
    return np.unique(np.concatenate(hit)) if hit else np.zeros(0, dtype=np.int64)


@dataclass
class DeviceProblem:
    """A case for device-resident stepping without the reference's host mesh arrays: the
    row-compact layout, boundary-condition / pin / reaction node sets, and (plain squares) the
    pre-crack segments for pf_init_state.  For the plain squares (config 5: 67 M cells) nothing
    of size n_elems is built on the host."""

    case: LoadCase
    layout: object
    params: object
    config: object
    bcs: list
    pins: object
    reactions: list
    boundary_sets: dict
    mesh: object = None   # the host mesh (non-plain cases only)


def device_problem(case: LoadCase, api=None) -> DeviceProblem:
    from types import SimpleNamespace  # noqa: PLC0415

    from .meshing import StructuredLayout  # noqa: PLC0415

    api = api or b200_api()
    params = material(case, api)
    config = api.SolverConfig(tol_st=case.tol_st)
    mesh = None
    if case.mesh[0] == "notched" and not case.mesh[4]:
        _, nx, ny, side, _ = case.mesh
        lay = StructuredLayout.rectangle(nx, ny, side / nx, side / ny)
        rows = np.arange(ny + 1, dtype=np.int64) * (nx + 1)
        cols = np.arange(nx + 1, dtype=np.int64)
        bsets = {"bottom": cols, "top": ny * (nx + 1) + cols, "left": rows, "right": rows + nx}
    else:
        mesh = build_mesh(case, api)
        lay = StructuredLayout.from_mesh(mesh)
        bsets = mesh.boundary_sets
    view = SimpleNamespace(boundary_sets=bsets)
    return DeviceProblem(case, lay, params, config, boundary_conditions(case, view),
                         pinned_nodes(case, view), reaction_sets(case, view), bsets, mesh)


@dataclass
class Problem:
    case: LoadCase
    api: object
    mesh: object
    disc: object
    params: object
    config: object
    state: object
    bcs: list
    pins: object
    reactions: list
    setup_s: float = 0.0


def setup(case: LoadCase, api, lin_method: str | None = None) -> Problem:
    t0 = time.perf_counter()
    mesh = build_mesh(case, api)
    disc = api.Discretization(mesh)
    params = material(case, api)
    cfg_kw = {"tol_st": case.tol_st}
    if lin_method is not None:
        cfg_kw["lin_method"] = lin_method
    config = api.SolverConfig(**cfg_kw)
    state = api.SolverState.zeros(disc)
    cracked = precrack_nodes(case, mesh)
    if cracked.size:
        state.d[cracked] = 1.0
        state.d_prev[cracked] = 1.0
    return Problem(case, api, mesh, disc, params, config, state,
                   boundary_conditions(case, mesh), pinned_nodes(case, mesh),
                   reaction_sets(case, mesh), time.perf_counter() - t0)


@dataclass
class StepRecord:
    step: int
    n_stag: int
    n_nr_u: int
    n_nr_d: int
    spd_fallbacks: int
    final_rd_ratio: float
    reactions: list = field(default_factory=list)
    wall: float = 0.0


def run(problem: Problem, scheme: str, n_steps: int | None = None, on_step=None,
        first_step: int = 1) -> list:
    """Advance ``n_steps`` load steps (default: the case's full schedule), numbering them from
    ``first_step`` (a restart from a saved state: every load step applies the same increment,
    so the number is only a label)."""
    api = problem.api
    kind = api.SchemeKind(scheme)
    n = problem.case.n_steps if n_steps is None else n_steps
    out = []
    for k in range(first_step, first_step + n):
        t0 = time.perf_counter()
        st = api.staggered_step(problem.disc, problem.state, kind, problem.bcs,
                                problem.params, problem.config, problem.pins)
        wall = time.perf_counter() - t0
        reac = [float(api.reaction_force(problem.disc, problem.state.u, problem.state.d,
                                         problem.params, nodes, comp))
                for _, nodes, comp in problem.reactions]
        rec = StepRecord(k, st.n_stag, st.n_nr_u, st.n_nr_d, st.spd_fallbacks,
                         float(st.final_rd_ratio), reac, wall)
        out.append(rec)
        if on_step is not None:
            on_step(rec, problem)
    return out
