"""Staggered iteration counts of the GPU solver around the crack step of a case, per scheme,
next to the reference's golden table (for the parity-band discussion in DESIGN.md section 4)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_07969_b200 import configs as C  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
schemes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["ST", "S1", "S2", "S3"]
for sch in schemes:
    z = np.load(os.path.join(ROOT, "tests", "golden", f"run_{case}_{sch}.npz"))
    ref = z["table"][:, 1].astype(int)
    pb = C.setup(C.get_case(case), C.b200_api())
    recs = C.run(pb, sch, n_steps=len(ref))
    got = np.array([r.n_stag for r in recs])
    diff = np.nonzero(got != ref)[0]
    print(f"{case} {sch}: total GPU {got.sum()} ref {ref.sum()}; differing steps "
          + ", ".join(f"{i + 1}: {got[i]} vs {ref[i]}" for i in diff), flush=True)
