"""Per-iteration cost of the persistent PCG kernels at every BASELINE.json mesh size.

Runs `pf_bench_cg` (a fixed number of PCG iterations, stopping test disabled) on the layouts
of cfg1..cfg5 with a seeded random state, so that the largest mesh (cfg5, 8192^2 cells,
67.1 M nodes / 134 M displacement DOFs) is measured without solving it to convergence.
Algorithmic bytes per iteration: momentum 168 B x N_nodes, phase field 72 B x N_nodes +
32 B x N_cells.  Prints one JSON line per case and physics.

usage: python scripts/roofline_sizes.py [cases...] [--iters N]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200 import meshing  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402


def layout_for(case):
    kind = case.mesh[0]
    if kind == "notched" and not case.mesh[4]:
        _, nx, ny, side, _ = case.mesh
        return meshing.StructuredLayout.rectangle(nx, ny, side / nx, side / ny)
    api = C.b200_api()
    return meshing.StructuredLayout.from_mesh(C.build_mesh(case, api))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["cfg1", "cfg2", "cfg4", "cfg3", "cfg5"])
    ap.add_argument("--iters", type=int, default=0, help="0: about 0.5 s per measurement")
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()

    mbw = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    peak = float(mbw.get("hbm_gbs", 0.0)) or None
    for name in args.cases:
        case = C.get_case(name)
        lay = layout_for(case)
        params = C.material(case, C.b200_api())
        config = C.b200_api().SolverConfig(tol_st=case.tol_st)
        s = DeviceSession(lay, params, config, device=0)
        rng = np.random.default_rng(7)
        nn, ne = lay.n_nodes, lay.n_elems
        s.push(u=1e-4 * rng.standard_normal(2 * nn), d=0.5 * rng.random(nn),
               d_prev=np.zeros(nn))
        s.refresh_gp()
        best_mom = None
        for phys, nbytes in (("momentum", 168.0 * nn), ("evolution", 72.0 * nn + 32.0 * ne)):
            n_iter = args.iters or max(20, int(0.5 / max(nbytes / 4.0e12, 1.2e-5)))
            s.flush_l2()
            s.bench_cg(phys, min(n_iter, 50))  # warm-up
            best = None
            # short launches: the well-conditioned phase-field system would otherwise drive r.r to an
            # exact zero (0/0 in beta) within a few hundred iterations
            chunk = min(n_iter, 2000 if phys == "momentum" else 100)
            for _r in range(args.repeats):
                tot_ms, tot_it = 0.0, 0
                while tot_it < n_iter:
                    s.flush_l2()
                    ms, it = s.bench_cg(phys, chunk)
                    tot_ms, tot_it = tot_ms + ms, tot_it + it
                us = 1e3 * tot_ms / tot_it
                best = us if best is None else min(best, us)
            gbs = nbytes / best / 1e3
            if phys == "momentum":
                best_mom = best
            print(json.dumps({
                "case": name, "physics": phys, "n_nodes": nn, "n_cells": ne,
                "iters": n_iter, "us_per_iter": round(best, 3),
                "algorithmic_bytes_per_iter": nbytes, "GBs": round(gbs, 1),
                "frac_of_measured_hbm": round(gbs / peak, 3) if peak else None,
                **s.device_info()}), flush=True)
        mg = s.mg_info()
        if mg["n_levels"]:  # multigrid momentum PCG: per-iteration cost and per-solve setup
            t = {}
            for n in (1, 11):
                s.flush_l2()
                s.bench_cg("momentum_mg", n)
                t[n] = min(s.bench_cg("momentum_mg", n)[0] for _ in range(args.repeats))
            per = (t[11] - t[1]) / 10.0
            print(json.dumps({
                "case": name, "physics": "momentum_mg", "n_nodes": nn, "levels": mg["n_levels"],
                "tail_from_level": mg["n_grid"], "us_per_iter": round(1e3 * per, 2),
                "setup_us": round(1e3 * (t[1] - per), 1),
                "jacobi_equivalent_iters": round(1e3 * per / best_mom, 1) if best_mom else None}),
                flush=True)
        s.close()


if __name__ == "__main__":
    main()
