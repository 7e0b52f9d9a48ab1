"""Round-off sensitivity of the reference ALGORITHM's per-step iteration counts.

At crack steps the staggered iteration count is chaotic: exact-arithmetic-equivalent
reformulations of the reference algorithm (different but equally valid floating-point
evaluation orders) change it by several iterations.  This script runs an ensemble of such
variants of the CPU oracle (oracle/phasefield_oracle.py, itself pinned to the unmodified
reference by tests/test_oracle_golden.py) on every golden case and records, per load step, the
n_stag of every variant.  tests/test_gpu_solver.py uses the spread as the "+-N where the
reference's own iterative tolerance allows" band of BASELINE.json's north star.

Variants (all mathematically identical to the reference):
  cg          the reference's own lin_method="cg" (Jacobi-PCG, rtol 1e-12)
  exact       exact uniform-cell geometry instead of coordinate-derived Jacobians
  exact_diff  exact geometry + strains from edge jumps (u1-u0) instead of B.u products
  pair        pairwise instead of sequential per-node accumulation
  gpu_like    exact + diff + element-Laplacian gradient term + pairwise + CG

    OMP_NUM_THREADS=1 python tests/golden/make_sensitivity.py tension16 ST
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

VARIANTS = {
    "cg": dict(lin_method="cg"),
    "exact": dict(geometry="exact"),
    "exact_diff": dict(geometry="exact", strain="differences"),
    "pair": dict(scatter="pairwise"),
    "gpu_like": dict(geometry="exact", strain="differences", gradterm="laplacian",
                     scatter="pairwise", lin_method="cg"),
}


def run_variant(case: str, scheme: str, variant: str, steps: int | None = None) -> list:
    pb = C.setup(C.get_case(case), oracle_api(**VARIANTS[variant]))
    return [r.n_stag for r in C.run(pb, scheme, n_steps=steps)]


def main() -> None:
    case, scheme = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else None
    t0 = time.time()
    out = {v: run_variant(case, scheme, v, steps) for v in VARIANTS}
    path = os.path.join(HERE, f"sens_{case}_{scheme}.json")
    with open(path, "w") as f:
        json.dump({"case": case, "scheme": scheme, "n_stag": out,
                   "seconds": round(time.time() - t0, 1)}, f)
    print("wrote", path, round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    main()
