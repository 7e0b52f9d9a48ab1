"""Per-step tables of the B200 path through the drop-in (the same runner as the reference's golden
tables, ``configs.run``): n_stag, n_nr_u, n_nr_d, spd_fallbacks, final ratio, reactions, plus
phase-field snapshots and restart states (u, d, d_prev, gp.psi_max) after selected steps.

    python scripts/gpu_tables.py CASE SCHEME [--steps N] [--snap 25,54] [--state-snap 54]
                                 [--restart FILE] [--out gpurun_out/tables/x.npz]

Solver variants are selected through the PFB200_* environment switches (read at pf_create).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from paper_2209_07969_b200 import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("scheme")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--snap", default="")
    ap.add_argument("--state-snap", default="")
    ap.add_argument("--restart", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    snaps = {int(x) for x in a.snap.split(",") if x}
    ssnaps = {int(x) for x in a.state_snap.split(",") if x}
    pb = C.setup(C.get_case(a.case), C.b200_api())
    first = 1
    if a.restart:
        from make_golden import load_restart  # noqa: PLC0415

        first = load_restart(pb.state, a.restart) + 1
    n = pb.case.n_steps - first + 1 if a.steps is None else a.steps
    out = a.out or os.path.join(ROOT, "gpurun_out", "tables", f"{a.case}_{a.scheme}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    rows, extra = [], {}
    t0 = time.perf_counter()

    def cb(rec, problem):
        rows.append([rec.step, rec.n_stag, rec.n_nr_u, rec.n_nr_d, rec.spd_fallbacks,
                     rec.final_rd_ratio, rec.wall] + list(rec.reactions))
        if rec.step in snaps:
            extra[f"d_step{rec.step}"] = problem.state.d.copy()
        if rec.step in ssnaps:
            st = problem.state
            np.savez_compressed(out.replace(".npz", f"_restart{rec.step}.npz"),
                                after_step=rec.step, u=st.u, d=st.d, d_prev=st.d_prev,
                                psi_max=st.gp.psi_max)

    C.run(pb, a.scheme, n_steps=n, on_step=cb, first_step=first)
    env = {k: v for k, v in os.environ.items() if k.startswith("PFB200_")}
    meta = dict(case=a.case, scheme=a.scheme, first_step=first, steps=len(rows), env=env,
                wall_s=time.perf_counter() - t0)
    np.savez_compressed(out, table=np.array(rows), meta=json.dumps(meta),
                        final_d=pb.state.d, **extra)
    tab = np.array(rows)
    print(json.dumps(dict(meta, total_n_stag=int(tab[:, 1].sum()),
                          n_stag=[int(x) for x in tab[:, 1]])), flush=True)


if __name__ == "__main__":
    main()
