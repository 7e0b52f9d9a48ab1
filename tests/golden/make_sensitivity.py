"""Round-off sensitivity of the reference ALGORITHM's per-step iteration counts.

At crack steps the staggered iteration count is chaotic: exact-arithmetic-equivalent
reformulations of the reference algorithm (different but equally valid floating-point
evaluation orders) change it by several iterations.  This script runs an ensemble of such
variants of the CPU oracle (oracle/phasefield_oracle.py, itself pinned to the unmodified
reference by tests/test_oracle_golden.py) on every golden case and records, per load step, the
n_stag of every variant.  tests/test_gpu_solver.py uses the spread as the "+-N where the
reference's own iterative tolerance allows" band of BASELINE.json's north star.

Variants: the full factorial of six exact-arithmetic-equivalent knobs (KNOBS below): geometry
from coordinates or exact constants, strains as B.u products or edge jumps, the phase-field
gradient term as gradient or element-Laplacian, per-node accumulation sequential or pairwise,
internal-force back-projection as one einsum or Gauss-point-pair grouped, and the linear
solver direct (SuperLU) or the reference's own lin_method="cg".  The crack side taken by the
symmetric tension test ("branch") is recorded too.

    OMP_NUM_THREADS=1 python tests/golden/make_sensitivity.py tension16 ST [steps|-] [max_variants|-] [a:b]
    OMP_NUM_THREADS=1 python tests/golden/make_sensitivity.py cfg1 ST - - exact:0:4   (exact-geometry half)
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.phasefield_oracle import oracle_api  # noqa: E402
from paper_2209_07969_b200 import configs as C  # noqa: E402

KNOBS = {
    "geometry": ("coords", "exact"),
    "strain": ("products", "differences"),
    "gradterm": ("gradient", "laplacian"),
    "scatter": ("sequential", "pairwise"),
    "backproj": ("einsum", "grouped"),
    "lin_method": ("direct", "cg"),
}


def factorial(max_variants: int | None = None) -> dict:
    """All non-default knob combinations (the default one is the pinned oracle itself)."""
    import itertools

    keys = list(KNOBS)
    out = {}
    for combo in itertools.product(*(range(len(KNOBS[k])) for k in keys)):
        if not any(combo):
            continue
        kw = {k: KNOBS[k][c] for k, c in zip(keys, combo) if c}
        out["+".join(f"{k}={v}" for k, v in kw.items())] = kw
    if max_variants is not None:  # deterministic thinning: keep every k-th combination
        names = list(out)
        step = max(1, len(names) // max_variants)
        out = {n: out[n] for n in names[::step][:max_variants]}
    return out


VARIANTS = factorial()


def run_variant(case: str, scheme: str, kw: dict, steps: int | None = None) -> tuple:
    pb = C.setup(C.get_case(case), oracle_api(**kw))
    stag = [r.n_stag for r in C.run(pb, scheme, n_steps=steps)]
    branch = None
    cs = C.get_case(case)
    if cs.loading == "tension" and cs.mesh[0] == "notched":
        n = cs.mesh[1]
        d = pb.state.d
        below = d[(n // 2 - 1) * (n + 1):(n // 2) * (n + 1)].mean()
        above = d[(n // 2 + 1) * (n + 1):(n // 2 + 2) * (n + 1)].mean()
        branch = "below" if below > above else ("above" if above > below else "symmetric")
    return stag, branch


def main() -> None:
    case, scheme = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
    maxv = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4] != "-" else None
    variants = factorial(maxv)
    suffix = ""
    if len(sys.argv) > 5:  # "a:b" slice of the full factorial, written to its own part file
        spec = sys.argv[5]
        full = factorial()
        if spec.startswith("exact:"):  # the exact-geometry half (uniform-cell constants, as
            spec = spec[len("exact:"):]  # the device path evaluates them)
            full = {n: kw for n, kw in full.items() if kw.get("geometry") == "exact"}
            suffix = "_exact"
        a, b = (int(x) for x in spec.split(":"))
        names = list(full)[a:b]
        variants = {n: full[n] for n in names}
        suffix += f"_part{a}_{b}"
    t0 = time.time()
    stag, branch = {}, {}
    for name, kw in variants.items():
        stag[name], branch[name] = run_variant(case, scheme, kw, steps)
    path = os.path.join(HERE, f"sens_{case}_{scheme}{suffix}.json")
    with open(path, "w") as f:
        json.dump({"case": case, "scheme": scheme, "n_stag": stag, "branch": branch,
                   "seconds": round(time.time() - t0, 1)}, f)
    print("wrote", path, round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    main()
