"""BASELINE configs[2] (1024^2 shear) at full size through its crack regime, device vs device:
the gated solves by the scalar multigrid PCG with the SPD probe inside (default) against the
Jacobi-PCG probe (PFB200_MGS_GATED=0).  Per-step staggered / Newton / fallback counts and the
reaction; the first load step whose counts differ, if any.

    python scripts/cfg3_gated_crosscheck.py [scheme] [n_steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

scheme = sys.argv[1] if len(sys.argv) > 1 else "S3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 120
dp = C.device_problem(C.get_case("cfg3"))
runs = {}
for gated in ("1", "0"):
    os.environ["PFB200_MGS_GATED"] = gated
    s = DeviceSession(dp.layout, dp.params, dp.config, device=0)
    s.init_state()
    rows, t0 = [], time.perf_counter()
    for k in range(steps):
        try:
            st = s.step(scheme, dp.bcs, dp.pins)
        except Exception as exc:  # noqa: BLE001  (e.g. the reference's max_stag limit)
            print(f"gated={gated}: load step {k + 1}: {type(exc).__name__}: {exc}", file=sys.stderr)
            break
        f = s.reaction_force(dp.reactions[0][1], dp.reactions[0][2])
        rows.append([st.n_stag, st.n_nr_u, st.n_nr_d, st.spd_fallbacks, f, int(st.cg_iters_d)])
        if time.perf_counter() - t0 > float(os.environ.get('XCHECK_BUDGET_S', '900')):
            break
    runs[gated] = rows
    s.close()
a, b = runs["1"], runs["0"]
n = min(len(a), len(b))
diff = next((k + 1 for k in range(n) if a[k][:4] != b[k][:4]), None)
fpeak = max(abs(r[4]) for r in b[:n])
out = {"case": "cfg3", "scheme": scheme, "steps_compared": n, "first_step_with_different_counts": diff,
       "n_stag_mg": [r[0] for r in a[:n]], "n_stag_jacobi": [r[0] for r in b[:n]],
       "fallbacks_mg": [r[3] for r in a[:n]], "fallbacks_jacobi": [r[3] for r in b[:n]],
       "max_force_diff_over_peak_before_diff": max(
           abs(a[k][4] - b[k][4]) for k in range(n if diff is None else diff - 1)) / fpeak,
       "pf_pcg_iterations": [sum(r[5] for r in a[:n]), sum(r[5] for r in b[:n])]}
print(json.dumps(out))
