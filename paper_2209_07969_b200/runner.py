"""Load-step runner and the SPEC output layout (the caller of the path).

The reference ships no runner (``pyproject.toml:16-17`` declares ``phasefrac.cli:main`` but
``cli.py`` is missing); its specification (``SPEC.md:401-471``, module ``bench_cli``) defines

* ``run`` — the time loop: per step apply the boundary increment, call ``staggered_step``,
  record the reaction and the iteration counts;
* ``write_csv`` — header ``time,u,reaction,n_stag,n_nr_u,n_nr_d``, one row per accepted step,
  decimal point, no locale (``SPEC.md:437``);
* ``write_vtk_snapshot`` — legacy-VTK ASCII: POINTS, CELLS, CELL_TYPES, POINT_DATA with the
  scalar ``d`` and the vector ``u`` (``SPEC.md:443-451``);
* ``sweep`` — the four schemes on one config, comparison CSV
  ``scheme,max_n_stag,total_n_stag,total_nr_u,total_nr_d,peak_force`` (``SPEC.md:465``).

The load cases are the named recipes of ``configs`` (BASELINE configs 1-5 and the reduced
analogues); a run config may override the increment, the step count and the outputs.  The
steps themselves go through the drop-in ``schemes.staggered_step`` (the B200 path) or, with
``api=oracle``, through any object exposing the reference's API (tests use the CPU oracle).

    python -m paper_2209_07969_b200.runner run --case tension16 --scheme S1 --out runs/t16
    python -m paper_2209_07969_b200.runner run --config my.ini
    python -m paper_2209_07969_b200.runner sweep --case tension16 --out runs/t16
"""

from __future__ import annotations

import argparse
import configparser
import csv
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import configs as C

CSV_HEADER = ("time", "u", "reaction", "n_stag", "n_nr_u", "n_nr_d")
SWEEP_HEADER = ("scheme", "max_n_stag", "total_n_stag", "total_nr_u", "total_nr_d", "peak_force")
SCHEMES = ("ST", "S1", "S2", "S3")


@dataclass
class ReportRow:
    time: float
    u: float
    reaction: float
    n_stag: int
    n_nr_u: int
    n_nr_d: int
    wall: float = 0.0


@dataclass
class RunReport:
    """Per-step rows and the Table-5 style totals (SPEC.md ``RunReport``)."""

    case: str
    scheme: str
    rows: list = field(default_factory=list)

    @property
    def max_n_stag(self) -> int:
        return max((r.n_stag for r in self.rows), default=0)

    @property
    def total_n_stag(self) -> int:
        return sum(r.n_stag for r in self.rows)

    @property
    def total_nr_u(self) -> int:
        return sum(r.n_nr_u for r in self.rows)

    @property
    def total_nr_d(self) -> int:
        return sum(r.n_nr_d for r in self.rows)

    @property
    def peak_force(self) -> float:
        return max((abs(r.reaction) for r in self.rows), default=0.0)


@dataclass
class RunConfig:
    case: str = "tension16"
    scheme: str = "S1"
    n_steps: int | None = None
    inc: float | None = None
    out: str | None = None
    vtk_every: int = 0  # 0: no snapshots; k: every k-th step and the last one


# ---- config files ---------------------------------------------------------------------------
_KEYS = {
    "problem": {"case": str, "scheme": str},
    "loading": {"steps": int, "increment": float},
    "output": {"dir": str, "vtk_every": int},
}


def parse_config(path: str) -> RunConfig:
    """Flat key-value config with sections ``[problem] [loading] [output]``.
    Unknown sections / keys and invalid values raise ``ValueError`` naming the line."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    lines = open(path).read().splitlines()

    def where(key):
        for k, ln in enumerate(lines, 1):
            if ln.strip().split("=")[0].strip() == key:
                return k
        return 0

    cp = configparser.ConfigParser()
    cp.read_string("\n".join(lines))
    cfg = RunConfig()
    for sec in cp.sections():
        if sec not in _KEYS:
            raise ValueError(f"{path}: unknown section [{sec}]")
        for key, raw in cp[sec].items():
            if key not in _KEYS[sec]:
                raise ValueError(f"{path}:{where(key)}: unknown key {key!r} in [{sec}]")
            try:
                val = _KEYS[sec][key](raw)
            except ValueError as exc:
                raise ValueError(f"{path}:{where(key)}: invalid value for {key}: {raw!r}") from exc
            if key == "case":
                if val not in C.CASES:
                    raise ValueError(f"{path}:{where(key)}: unknown case {val!r}")
                cfg.case = val
            elif key == "scheme":
                if val not in SCHEMES:
                    raise ValueError(f"{path}:{where(key)}: unknown scheme {val!r}")
                cfg.scheme = val
            elif key == "steps":
                if val < 0:
                    raise ValueError(f"{path}:{where(key)}: steps must be >= 0")
                cfg.n_steps = val
            elif key == "increment":
                if not val > 0.0:
                    raise ValueError(f"{path}:{where(key)}: increment must be > 0")
                cfg.inc = val
            elif key == "dir":
                cfg.out = val
            elif key == "vtk_every":
                cfg.vtk_every = max(0, val)
    return cfg


# ---- writers --------------------------------------------------------------------------------
def write_csv(report: RunReport, path: str) -> None:
    """``time,u,reaction,n_stag,n_nr_u,n_nr_d``; floats as ``repr`` (exact round trip)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r in report.rows:
            w.writerow((repr(float(r.time)), repr(float(r.u)), repr(float(r.reaction)),
                        int(r.n_stag), int(r.n_nr_u), int(r.n_nr_d)))


def read_csv(path: str) -> list:
    with open(path, newline="") as f:
        rd = csv.reader(f)
        header = next(rd)
        if tuple(header) != CSV_HEADER:
            raise ValueError(f"{path}: unexpected header {header}")
        return [ReportRow(float(t), float(u), float(fr), int(a), int(b), int(c))
                for t, u, fr, a, b, c in rd]


def write_sweep_csv(reports: list, path: str) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(SWEEP_HEADER)
        for rep in reports:
            w.writerow((rep.scheme, rep.max_n_stag, rep.total_n_stag, rep.total_nr_u,
                        rep.total_nr_d, repr(float(rep.peak_force))))


def write_vtk_snapshot(mesh, u, d, path: str, title: str = "phase-field snapshot") -> None:
    """Legacy-VTK ASCII unstructured grid of Q4 cells (VTK_QUAD = 9) with POINT_DATA ``d``
    (scalar) and ``u`` (vector, z = 0)."""
    nodes = np.asarray(mesh.nodes, dtype=np.float64)
    cells = np.asarray(mesh.elements, dtype=np.int64)
    u = np.asarray(u, dtype=np.float64).reshape(-1, 2)
    d = np.asarray(d, dtype=np.float64).ravel()
    n, ne = nodes.shape[0], cells.shape[0]
    if u.shape[0] != n or d.shape[0] != n:
        raise ValueError("fields must be sized to the mesh nodes")
    with open(path, "w") as f:
        f.write("# vtk DataFile Version 3.0\n")
        f.write(title.replace("\n", " ")[:255] + "\n")
        f.write("ASCII\nDATASET UNSTRUCTURED_GRID\n")
        f.write(f"POINTS {n} double\n")
        for x, y in nodes.tolist():
            f.write(f"{x!r} {y!r} 0.0\n")
        f.write(f"CELLS {ne} {5 * ne}\n")
        for c in cells.tolist():
            f.write(f"4 {c[0]} {c[1]} {c[2]} {c[3]}\n")
        f.write(f"CELL_TYPES {ne}\n")
        f.write("9\n" * ne)
        f.write(f"POINT_DATA {n}\nSCALARS d double 1\nLOOKUP_TABLE default\n")
        for v in d.tolist():
            f.write(f"{v!r}\n")
        f.write("VECTORS u double\n")
        for ux, uy in u.tolist():
            f.write(f"{ux!r} {uy!r} 0.0\n")


# ---- the time loop ---------------------------------------------------------------------------
def run_benchmark(cfg: RunConfig, api=None, on_step=None) -> RunReport:
    """Set up the case, advance its load steps through ``staggered_step`` and record one row per
    step: pseudo-time = step index, u = applied boundary displacement, reaction = the case's
    first reaction set (N per unit thickness).  Writes ``<out>/<case>_<scheme>.csv`` and VTK
    snapshots when ``cfg.out`` is set.  Solver errors propagate annotated with the step."""
    api = api or C.b200_api()
    overrides = {}
    if cfg.inc is not None:
        overrides["inc"] = cfg.inc
    if cfg.n_steps is not None:
        overrides["n_steps"] = cfg.n_steps
    case = C.get_case(cfg.case, **overrides)
    pb = C.setup(case, api)
    kind = api.SchemeKind(cfg.scheme)
    rep = RunReport(case.name, cfg.scheme)
    if cfg.out:
        os.makedirs(cfg.out, exist_ok=True)
    label, nodes, comp = pb.reactions[0]
    for k in range(1, case.n_steps + 1):
        t0 = time.perf_counter()
        try:
            st = api.staggered_step(pb.disc, pb.state, kind, pb.bcs, pb.params, pb.config,
                                    pb.pins)
        except Exception as exc:  # annotate the failing step (SPEC.md run_benchmark errors)
            exc.args = (f"load step {k} of {case.name} ({cfg.scheme}): {exc.args[0] if exc.args else exc}",
                        *exc.args[1:])
            raise
        wall = time.perf_counter() - t0
        f = float(api.reaction_force(pb.disc, pb.state.u, pb.state.d, pb.params, nodes, comp))
        row = ReportRow(float(k), k * case.inc, f, int(st.n_stag), int(st.n_nr_u),
                        int(st.n_nr_d), wall)
        rep.rows.append(row)
        if on_step is not None:
            on_step(row, pb)
        if cfg.out and cfg.vtk_every and (k % cfg.vtk_every == 0 or k == case.n_steps):
            write_vtk_snapshot(pb.mesh, pb.state.u, pb.state.d,
                               os.path.join(cfg.out, f"{case.name}_{cfg.scheme}_{k:05d}.vtk"),
                               f"{case.name} {cfg.scheme} step {k}")
    if cfg.out:
        write_csv(rep, os.path.join(cfg.out, f"{case.name}_{cfg.scheme}.csv"))
    return rep


def sweep(cfg: RunConfig, schemes=SCHEMES, api=None) -> list:
    """The given schemes on one config; writes ``<out>/<case>_sweep.csv``."""
    reports = []
    for sch in schemes:
        sub = RunConfig(cfg.case, sch, cfg.n_steps, cfg.inc, cfg.out, cfg.vtk_every)
        reports.append(run_benchmark(sub, api))
    if cfg.out:
        write_sweep_csv(reports, os.path.join(cfg.out, f"{cfg.case}_sweep.csv"))
    return reports


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2209_07969_b200.runner")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        p.add_argument("--case")
        p.add_argument("--scheme", choices=SCHEMES)
        p.add_argument("--steps", type=int)
        p.add_argument("--out")
        p.add_argument("--vtk-every", type=int)
    a = ap.parse_args(argv)
    cfg = parse_config(a.config) if a.config else RunConfig()
    cfg.case = a.case or cfg.case
    cfg.scheme = a.scheme or cfg.scheme
    cfg.n_steps = a.steps if a.steps is not None else cfg.n_steps
    cfg.out = a.out or cfg.out
    cfg.vtk_every = a.vtk_every if a.vtk_every is not None else cfg.vtk_every
    if a.cmd == "run":
        rep = run_benchmark(cfg)
        print(f"{rep.case} {rep.scheme}: {len(rep.rows)} steps, total n_stag {rep.total_n_stag}, "
              f"peak force {rep.peak_force:.6g}")
    else:
        for rep in sweep(cfg):
            print(f"{rep.case} {rep.scheme}: max n_stag {rep.max_n_stag}, total "
                  f"{rep.total_n_stag}, peak force {rep.peak_force:.6g}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
