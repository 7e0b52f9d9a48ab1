"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference at /root/reference does not exist on the GPU
box; the fixtures it writes are committed and travel instead):

    OMP_NUM_THREADS=1 python tests/golden/make_golden.py kat
    OMP_NUM_THREADS=1 python tests/golden/make_golden.py run tension16 ST
    OMP_NUM_THREADS=1 python tests/golden/make_golden.py run cfg1 S1 --snap 10,40,60,64,65
    OMP_NUM_THREADS=1 python tests/golden/make_golden.py run cfg2 ST --steps 2
    OMP_NUM_THREADS=1 python tests/golden/make_golden.py spd tension16 S1
    OMP_NUM_THREADS=1 python tests/golden/make_golden.py bar

Outputs (``tests/golden/``):
  * ``kat_<mesh>.npz``   — seeded random states and the reference's assembled residuals,
    tangent-vector products, diagonals, GP refresh, gate / extra stiffness / energy update,
    internal force, reaction force and evolution residual norm (pins the oracle and the
    GPU kernels);
  * ``run_<case>_<scheme>.npz`` — per-step table (n_stag, n_nr_u, n_nr_d, spd_fallbacks,
    final_rd_ratio, reactions) plus state snapshots (end-to-end parity);
  * ``spd_<case>_<scheme>.npz`` — states at which ``check_spd`` was called during a run and
    its decision (the SPD-predicate agreement test, SURVEY.md §7 hard part 1).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from paper_2209_07969_b200 import configs as C  # noqa: E402

REF_SRC = "/root/reference/pkg/src"


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from phasefrac import assembly, linsolve, material, meshing, schemes

    return assembly, linsolve, material, meshing, schemes


# -------------------------------------------------------------------------------------------
def kat(only=None) -> None:
    """Kernel-level known answers on small meshes from seeded random states."""
    assembly, linsolve, material, meshing, schemes = _ref()
    meshes = {
        "notched8": lambda: meshing.build_notched_square(8, 8, 1.0),
        "notched12x6": lambda: meshing.build_notched_square(12, 6, 2.0),
        "plain10": lambda: meshing.build_notched_square(10, 10, 1000.0, False),
        "lshape": lambda: meshing.build_lshape_mesh(62.5),
        # slit row on a tile boundary (TY = 8) and a slit spanning two tile columns (TX = 32)
        "notched16": lambda: meshing.build_notched_square(16, 16, 1.0),
        "notched80x16": lambda: meshing.build_notched_square(80, 16, 5.0),
        "lshape12p5": lambda: meshing.build_lshape_mesh(12.5),
    }
    params = material.MaterialParams.from_young_poisson(
        210000.0, 0.3, g_c=2.7, length_l=0.05, at_model="AT2")
    params_at1 = material.MaterialParams.from_young_poisson(
        210000.0, 0.3, g_c=2.7, length_l=0.05, at_model="AT1")
    for name, build in meshes.items():
        if only and name not in only:
            continue
        rng = np.random.default_rng(1234)
        mesh = build()
        disc = assembly.Discretization(mesh)
        nn, ne = mesh.n_nodes, mesh.n_elems
        scale = 1e-3 * float(np.ptp(mesh.nodes[:, 0]))
        u = rng.standard_normal(2 * nn) * scale
        d = rng.uniform(0.0, 0.9, nn)
        d_prev = np.clip(d - rng.uniform(-0.05, 0.1, nn), 0.0, None)
        xu = rng.standard_normal(2 * nn)
        xd = rng.standard_normal(nn)
        out = dict(nodes=mesh.nodes, elements=mesh.elements, u=u, d=d, d_prev=d_prev,
                   xu=xu, xd=xd)
        for tag, pr in (("at2", params), ("at1", params_at1)):
            sysm = assembly.assemble_momentum(disc, u, d, pr)
            out[f"{tag}_mom_R"] = sysm.residual
            out[f"{tag}_mom_Kx"] = sysm.stiffness @ xu
            out[f"{tag}_mom_diag"] = sysm.stiffness.diagonal()
            gp = assembly.GaussPointState.zeros(ne, 4)
            assembly.refresh_gp_from_displacement(disc, gp, u, pr)
            out[f"{tag}_gp_tr"] = gp.tr_eps
            out[f"{tag}_gp_trp"] = gp.tr_eps_plus
            out[f"{tag}_gp_dev2"] = gp.dev_dot_dev
            out[f"{tag}_gp_psi"] = gp.psi_plus
            out[f"{tag}_gp_strain"] = gp.strain
            # psi_max: a random history below/above the current energy
            gp.psi_max = gp.psi_plus * rng.uniform(0.5, 1.5, gp.psi_plus.shape)
            out[f"{tag}_gp_psimax"] = gp.psi_max
            ev = assembly.assemble_evolution(disc, d, d_prev, gp, pr)
            out[f"{tag}_evo_R"] = ev.residual
            out[f"{tag}_evo_Kx"] = ev.stiffness @ xd
            out[f"{tag}_evo_diag"] = ev.stiffness.diagonal()
            d_gp = disc.interp_nodal(d)
            out[f"{tag}_gate"] = schemes.softening_gate(gp, d_gp, pr, 0.95)
            dd = rng.standard_normal(nn) * 0.05
            out[f"{tag}_dd"] = dd
            for sk in ("S1", "S2", "S3"):
                kind = schemes.SchemeKind(sk)
                extra = schemes.extra_stiffness(kind, gp, d_gp, pr, 0.95)
                out[f"{tag}_{sk}_extra"] = extra
                ev2 = assembly.assemble_evolution(disc, d, d_prev, gp, pr, scheme_extra=extra)
                out[f"{tag}_{sk}_evo_Kx"] = ev2.stiffness @ xd
                out[f"{tag}_{sk}_evo_diag"] = ev2.stiffness.diagonal()
                gate = schemes.softening_gate(gp, d_gp, pr, 0.95)
                trp, dev2, psi = schemes.update_active_energy(
                    kind, gp, disc.interp_nodal(dd), d_gp, pr, gate)
                out[f"{tag}_{sk}_upd_trp"] = trp
                out[f"{tag}_{sk}_upd_dev2"] = dev2
                out[f"{tag}_{sk}_upd_psi"] = psi
            out[f"{tag}_fint"] = assembly.internal_force(disc, u, d, pr)
            bsets = mesh.boundary_sets
            key = "top" if "top" in bsets else "load_zone"
            out[f"{tag}_reac_{key}_1"] = np.array(
                assembly.reaction_force(disc, u, d, pr, bsets[key], 1))
            st = schemes.SolverState(u=u.copy(), d=d.copy(), d_prev=d_prev.copy(), gp=gp)
            out[f"{tag}_evo_norm"] = np.array(schemes.evolution_residual_norm(disc, st, pr))
        path = os.path.join(HERE, f"kat_{name}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, flush=True)


# -------------------------------------------------------------------------------------------
def _state_arrays(state) -> dict:
    gp = state.gp
    return dict(u=state.u.copy(), d=state.d.copy(), d_prev=state.d_prev.copy(),
                tr_eps_plus=gp.tr_eps_plus.copy(), dev_dot_dev=gp.dev_dot_dev.copy(),
                psi_plus=gp.psi_plus.copy(), psi_max=gp.psi_max.copy())


def restart_state_arrays(state) -> dict:
    """The part of a SolverState that determines the next load step: u, d, d_prev and
    gp.psi_max.  The other GP arrays are overwritten from u by the k = 0 momentum pass
    (``schemes.py:237`` -> ``assembly.py:260-269``) before anything reads them."""
    return dict(u=state.u.copy(), d=state.d.copy(), d_prev=state.d_prev.copy(),
                psi_max=state.gp.psi_max.copy())


def load_restart(state, path: str) -> int:
    """Overwrite ``state`` with a restart file; returns the load step it was taken after."""
    z = np.load(path)
    state.u[:] = z["u"]
    state.d[:] = z["d"]
    state.d_prev = z["d_prev"].copy()
    state.gp.psi_max = z["psi_max"].copy()
    return int(z["after_step"])


def run(case_name: str, scheme: str, steps: int | None, snaps: list[int],
        lin_method: str | None, partial: bool = False, state_snaps: tuple = (),
        restart: str | None = None, tag_extra: str = "") -> None:
    """Run the reference on a case.  ``partial``: rewrite the output after every load step
    (long full-size runs, meta["complete"] tells whether the run finished).  ``state_snaps``:
    also store the restart state after those steps (``restart_step<k>.npz``).  ``restart``:
    start from such a restart file (the reference crack step from a given state)."""
    api = C.reference_api(REF_SRC)
    case = C.get_case(case_name)
    pb = C.setup(case, api, lin_method=lin_method)
    first = 1
    if restart:
        first = load_restart(pb.state, restart) + 1
    n = case.n_steps - first + 1 if steps is None else steps
    rows, snap = [], {}
    t_loop = 0.0
    suffix = "" if lin_method in (None, "direct") else f"_{lin_method}"
    tag = (f"{case_name}_{scheme}{suffix}{tag_extra}"
           + ("" if steps is None or partial else f"_{n}steps"))
    path = os.path.join(HERE, f"run_{tag}.npz")

    def meta(complete):
        return dict(case=case_name, scheme=scheme, steps=len(rows), first_step=first,
                    complete=complete, restart=os.path.basename(restart) if restart else None,
                    lin_method=lin_method or "direct",
                    loop_wall_s=t_loop, n_nodes=int(pb.mesh.n_nodes),
                    n_elems=int(pb.mesh.n_elems),
                    columns=["step", "n_stag", "n_nr_u", "n_nr_d", "spd_fallbacks",
                             "final_rd_ratio", "wall"] + [r[0] for r in pb.reactions],
                    generator="tests/golden/make_golden.py (unmodified reference, "
                              "/root/reference/pkg/src/phasefrac)")

    def write(complete):
        final = _state_arrays(pb.state) if pb.mesh.n_nodes <= 20000 else {
            "d": pb.state.d.copy(), "u": pb.state.u.copy()}
        tmp = path + ".tmp.npz"
        np.savez_compressed(tmp, table=np.array(rows), meta=json.dumps(meta(complete)),
                            **{f"final_{k}": v for k, v in final.items()}, **snap)
        os.replace(tmp, path)

    def cb(rec, problem):
        nonlocal t_loop
        t_loop += rec.wall
        rows.append([rec.step, rec.n_stag, rec.n_nr_u, rec.n_nr_d, rec.spd_fallbacks,
                     rec.final_rd_ratio, rec.wall] + list(rec.reactions))
        print(case_name, scheme, rows[-1], flush=True)
        if rec.step in snaps:
            snap[f"d_step{rec.step}"] = problem.state.d.copy()
            snap[f"u_step{rec.step}"] = problem.state.u.copy()
        if rec.step in state_snaps:
            rp = os.path.join(HERE, f"restart_{case_name}_{scheme}_step{rec.step}.npz")
            np.savez_compressed(rp, after_step=rec.step, **restart_state_arrays(problem.state))
            print("wrote", rp, flush=True)
        if partial:
            write(False)

    C.run(pb, scheme, n_steps=n, on_step=cb, first_step=first)
    write(True)
    print("wrote", path, "loop", round(t_loop, 1), "s", flush=True)


# -------------------------------------------------------------------------------------------
def spd(case_name: str, scheme: str, max_each: int) -> None:
    """Record states at check_spd calls and the reference decision."""
    assembly, linsolve, material, meshing, schemes = _ref()
    api = C.reference_api(REF_SRC)
    case = C.get_case(case_name)
    pb = C.setup(case, api)
    recs = {"fallback": [], "spd": []}
    orig = schemes.check_spd
    counter = {"calls": 0}

    def wrapped(matrix):
        val = orig(matrix)
        counter["calls"] += 1
        key = "fallback" if val <= 0.0 else "spd"
        if len(recs[key]) < max_each:
            s = pb.state
            recs[key].append(dict(
                d=s.d.copy(), d_prev=s.d_prev.copy(), trp=s.gp.tr_eps_plus.copy(),
                dev2=s.gp.dev_dot_dev.copy(), psi=s.gp.psi_plus.copy(),
                psimax=s.gp.psi_max.copy(), pivot=val))
        return val

    schemes.check_spd = wrapped
    try:
        C.run(pb, scheme)
    finally:
        schemes.check_spd = orig
    out = {}
    for key, lst in recs.items():
        for i, r in enumerate(lst):
            for k, v in r.items():
                out[f"{key}{i}_{k}"] = np.asarray(v)
    out["meta"] = json.dumps(dict(case=case_name, scheme=scheme, calls=counter["calls"],
                                  n_fallback=len(recs["fallback"]), n_spd=len(recs["spd"])))
    path = os.path.join(HERE, f"spd_{case_name}_{scheme}.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, counter, flush=True)


def bar() -> None:
    """The localizing bar of SPEC.md Appendix C (oracle/bar_analytic.py) on the unmodified
    reference: per-step staggered counts and the final phase field per scheme."""
    from oracle import bar_analytic as B

    api = C.reference_api(REF_SRC)
    out = {}
    for scheme in ("ST", "S1", "S3"):
        counts, k, d = B.run_localizing_bar(api, scheme)
        out[f"{scheme}_n_stag"] = np.array(counts)
        out[f"{scheme}_crack_step"] = np.array(k)
        out[f"{scheme}_d"] = d
        print("bar", scheme, "crack step", k, "n_stag", counts[k], flush=True)
    path = os.path.join(HERE, "bar_localizing.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


def main() -> None:
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    k = sub.add_parser("kat")
    k.add_argument("only", nargs="*")
    r = sub.add_parser("run")
    r.add_argument("case")
    r.add_argument("scheme")
    r.add_argument("--steps", type=int, default=None)
    r.add_argument("--snap", default="")
    r.add_argument("--lin", default=None)
    r.add_argument("--partial", action="store_true")
    r.add_argument("--state-snap", default="")
    r.add_argument("--restart", default=None)
    r.add_argument("--tag", default="")
    sub.add_parser("bar")
    s = sub.add_parser("spd")
    s.add_argument("case")
    s.add_argument("scheme")
    s.add_argument("--max-each", type=int, default=12)
    a = ap.parse_args()
    t0 = time.time()
    if a.cmd == "kat":
        kat(a.only)
    elif a.cmd == "bar":
        bar()
    elif a.cmd == "run":
        snaps = [int(x) for x in a.snap.split(",") if x]
        run(a.case, a.scheme, a.steps, snaps, a.lin, a.partial,
            tuple(int(x) for x in a.state_snap.split(",") if x), a.restart, a.tag)
    else:
        spd(a.case, a.scheme, a.max_each)
    print("elapsed", round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    main()
